// gspn_stream.cu — the TMA-streaming fast path for sm_100a (B200).
//
// One persistent launch covers every requested direction (PAPER.md:122-123 "Kernel Fuse", :201 — the
// paper's one-stream-per-direction concurrency becomes a direction dimension of the work queue).
// Work item = one chain (direction k, batch b, channel c): a P-wide state marching L steps. A CTA owns
// a chain at a time: warp NWC (the producer) streams K-step tiles of every input tensor into a
// shared-memory ring with TMA (cp.async.bulk.tensor, mbarrier complete_tx), NWC consumer warps run
// the recurrence with the carry in fp32 registers, exchange neighbours with warp shuffles and, across
// warps, through a shared-memory halo (one named barrier per step), and stage outputs in shared
// memory for TMA stores. Loads are 16-byte vectors from shared memory in both orientations:
//   T2B/B2T (vertical):   a tile is K image rows x P columns ([box][K][BW] in SMEM); a lane owns
//                         E = 4 consecutive positions and reads one 4-element vector per step.
//   L2R/R2L (horizontal): a tile is P image rows x K columns ([P][K], 16-byte rows = K steps); a lane
//                         owns NS = 4 interleaved rows and reads all K steps of a row in one vector.
// The chain order puts the D directions of one (b, c) plane next to each other so the plane's x (and
// in bwd the fp32 dx accumulator) is shared through L2 by co-scheduled CTAs.
//
// Backward: tiles in reverse step order; g_t = dh_t + b_{t+1} g_{t+1}
// + a_{t+1}[r+1] g_{t+1}[r+1] + c_{t+1}[r-1] g_{t+1}[r-1] exchanged as (a g, c g) products; h_{t-1}
// comes from a second TMA view of h shifted by one step (its zero fill at t = 0 is h_{-1} = 0);
// dx (sum over directions) accumulates with red.global.add.v4.f32 into an fp32 workspace plane and is
// converted by the last of the plane's D chains; per-channel dw gets the normalisation Jacobian in
// registers; grouped dw accumulates the normalised-tap gradients in fp32 and the group's last
// channel applies the Jacobian.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "gspn_common.cuh"
#include "gspn_internal.h"

namespace gspn {
namespace {

constexpr int kE = 2;        // vertical: consecutive positions per lane
constexpr int kNS = 2;       // horizontal: interleaved rows per lane
constexpr int kLanePos = 32 * kE;  // positions per consumer warp (both orientations: 32*kNS == 32*kE)
constexpr int kHaloW = 16;   // halo slots (>= consumer warps of any instantiation)
constexpr int kMaxIn = 7;
constexpr int kMaxOut = 4;
constexpr int kBarStep = 1;  // named barrier ids (0 is __syncthreads)
constexpr int kBarTile = 2;

struct Plan {
  int K;               // steps per tile: K * sizeof(T) == 16 bytes
  int nwc;             // consumer warps
  int ppad;            // positions covered: kLanePos * nwc
  int es;              // element size in bytes
  int bw, nbw;         // vertical TMA box width (positions) and box count
  int bh, nbh;         // horizontal TMA box height (positions) and box count
  int nin, nout;       // input / output tensors per tile
  int nstages;
  uint32_t tile_bytes;   // one tensor's tile in SMEM: K * ppad * es (= 16 * ppad)
  uint32_t stage_bytes;  // (nin + h_wide) * tile_bytes
  int h_wide;            // bwd: the h slot (last input) holds 2K steps for horizontal chains
  uint32_t out_bytes;    // nout * tile_bytes (one staging buffer; two are allocated)
  uint32_t tx_v, tx_h;   // TMA bytes landing per stage (vertical / horizontal chains)
  int64_t nchains;
  uint32_t smem_bytes;
};

struct alignas(64) StreamArgs {
  CUtensorMap in[2][kMaxIn];    // [0 vertical | 1 horizontal][tensor]
  CUtensorMap out[2][kMaxOut];
  ScanParams p;
  Plan plan;
};

// ------------------------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "WAIT%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_store3(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2,
                                           uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void red_add_v2(float* p, float a, float b, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(a), "f"(b), "l"(pol) : "memory");
}

__device__ __forceinline__ void red_add_f32(float* p, float a, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(a), "l"(pol) : "memory");
}

__device__ __forceinline__ float fast_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// ------------------------------------------------------------------------------ element access

// 2 consecutive elements of T at a shared-memory address <-> floats (4 B for bf16, 8 B for fp32).
template <typename T> struct V2;
template <> struct V2<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const uint8_t* p, float (&v)[2]) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
    v[0] = __uint_as_float(u << 16);
    v[1] = __uint_as_float(u & 0xFFFF0000u);
  }
  static __device__ __forceinline__ void store(uint8_t* p, const float (&v)[2]) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
    *reinterpret_cast<__nv_bfloat162*>(p) = a;
  }
};
template <> struct V2<float> {
  static __device__ __forceinline__ void load(const uint8_t* p, float (&v)[2]) {
    const float2 u = *reinterpret_cast<const float2*>(p);
    v[0] = u.x;
    v[1] = u.y;
  }
  static __device__ __forceinline__ void store(uint8_t* p, const float (&v)[2]) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  }
};

// 4 consecutive elements from fp32 -> T in global memory (dx conversion).
template <typename T> __device__ __forceinline__ void store4(T* p, float4 v);
template <> __device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* p, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}
template <> __device__ __forceinline__ void store4<float>(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

// One 16-byte row chunk = K steps of one position (horizontal tiles). Indices are compile-time
// constants after unrolling, so the selects fold away.
template <typename T> struct Row;
template <> struct Row<__nv_bfloat16> {
  static constexpr int K = 8;
  static __device__ __forceinline__ float get(const uint4& u, int i) {
    const uint32_t w = (i < 2) ? u.x : (i < 4) ? u.y : (i < 6) ? u.z : u.w;
    return (i & 1) ? __uint_as_float(w & 0xFFFF0000u) : __uint_as_float(w << 16);
  }
  static __device__ __forceinline__ void set(uint4& u, int i, float v) {
    const uint32_t b = static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v)));
    uint32_t& w = (i < 2) ? u.x : (i < 4) ? u.y : (i < 6) ? u.z : u.w;
    w = (i & 1) ? ((w & 0x0000FFFFu) | (b << 16)) : ((w & 0xFFFF0000u) | b);
  }
};
template <> struct Row<float> {
  static constexpr int K = 4;
  static __device__ __forceinline__ float get(const uint4& u, int i) {
    return __uint_as_float((i == 0) ? u.x : (i == 1) ? u.y : (i == 2) ? u.z : u.w);
  }
  static __device__ __forceinline__ void set(uint4& u, int i, float v) {
    uint32_t& w = (i == 0) ? u.x : (i == 1) ? u.y : (i == 2) ? u.z : u.w;
    w = __float_as_uint(v);
  }
};

// Shared-memory byte offset of (step-in-tile kk, position r) inside one vertical tensor tile
// ([box][K][bw] as written by the TMA boxes). Horizontal tiles are [position][16 bytes].
struct TileGeom {
  int K, bw_log2, es;
  __device__ __forceinline__ uint32_t vert(int kk, int r) const {
    const int bw = 1 << bw_log2;
    return static_cast<uint32_t>((((r >> bw_log2) * K + kk) * bw + (r & (bw - 1))) * es);
  }
};

// ------------------------------------------------------------------------------ chain bookkeeping

struct Chain {
  int k;            // direction slab
  uint32_t dir;
  bool vert, rev;   // orientation; reversed step order in canonical coordinates (B2T, R2L)
  int64_t bc, b, c, g, chain, wplane;
  int L, P, ntiles;
};

__device__ __forceinline__ Chain make_chain(const ScanParams& p, int K, int64_t w) {
  Chain ch;
  const int64_t bc = w / p.D;
  ch.k = static_cast<int>(w % p.D);
  ch.dir = p.dirbit[ch.k];
  ch.vert = (ch.dir == GSPN_DIR_T2B) || (ch.dir == GSPN_DIR_B2T);
  ch.rev = (ch.dir == GSPN_DIR_B2T) || (ch.dir == GSPN_DIR_R2L);
  ch.bc = bc;
  ch.b = bc / p.C;
  ch.c = bc % p.C;
  ch.g = ch.c / (p.C / p.G);
  ch.chain = (ch.k * p.B + ch.b) * p.C + ch.c;
  ch.wplane = (ch.k * p.B + ch.b) * p.G + ch.g;
  ch.L = static_cast<int>(ch.vert ? p.H : p.W);
  ch.P = static_cast<int>(ch.vert ? p.W : p.H);
  ch.ntiles = (ch.L + K - 1) / K;
  return ch;
}

// Canonical start coordinate (row for vertical, column for horizontal) of tile j.
__device__ __forceinline__ int tile_start(const Chain& ch, int j, int K) {
  return ch.rev ? (ch.L - (j + 1) * K) : (j * K);
}

// Input tensor slots.
enum FwdIn { F_X = 0, F_LAM, F_WL, F_WM, F_WR, F_NIN };
enum BwdIn { B_X = 0, B_LAM, B_DH, B_WL, B_WM, B_WR, B_H, B_NIN };
enum BwdOut { O_DLAM = 0, O_DWL, O_DWM, O_DWR };

template <bool kBwd>
__device__ __forceinline__ int64_t plane_of(const Chain& ch, int slot) {
  const bool is_x = kBwd ? (slot == B_X) : (slot == F_X);
  const bool is_w = kBwd ? (slot == B_WL || slot == B_WM || slot == B_WR) : (slot == F_WL || slot == F_WM || slot == F_WR);
  return is_x ? ch.bc : (is_w ? ch.wplane : ch.chain);
}

// ------------------------------------------------------------------------------ producer

template <bool kBwd>
__device__ void producer_loop(const StreamArgs& A, uint8_t* ring, uint64_t* full, uint64_t* empty) {
  const Plan& pl = A.plan;
  const ScanParams& p = A.p;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_normal();
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t w = blockIdx.x; w < pl.nchains; w += gridDim.x) {
    const Chain ch = make_chain(p, pl.K, w);
    const int o = ch.vert ? 0 : 1;
    for (int jj = 0; jj < ch.ntiles; ++jj) {
      const int j = kBwd ? (ch.ntiles - 1 - jj) : jj;
      mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
      const uint32_t fb = smem_u32(&full[stage]);
      mbar_arrive_tx(fb, ch.vert ? pl.tx_v : pl.tx_h);
      const int s0 = tile_start(ch, j, pl.K);
      const uint32_t st = smem_u32(ring + static_cast<size_t>(stage) * pl.stage_bytes);
      for (int t = 0; t < pl.nin; ++t) {
        const int plane = static_cast<int>(plane_of<kBwd>(ch, t));
        // h_{t-1} view for the backward, one step against the scan direction (its zero fill is
        // h_{-1} = 0). Vertical: the row coordinate shifts by one. Horizontal: TMA needs a 16-byte
        // aligned inner coordinate, so a 2K-step box [s0-K, s0+K) (L2R) / [s0, s0+2K) (R2L) is loaded
        // with a 32-byte swizzle and the consumer picks element K+kk-1 / kk+1.
        const bool hview = kBwd && t == B_H;
        const int shift = (hview && ch.vert) ? (ch.rev ? 1 : -1) : 0;
        // x is re-read by the plane's other directions; horizontal 16-byte row chunks are re-read
        // by the next tiles through the 128-byte L2 promotion: keep those at normal priority.
        const uint64_t pol = (t == 0 || !ch.vert) ? pol_keep : pol_stream;
        const uint32_t dst = st + t * pl.tile_bytes;
        if (ch.vert) {
          for (int q = 0; q < pl.nbw; ++q)
            tma_load3(dst + q * pl.K * pl.bw * pl.es, &A.in[o][t], q * pl.bw, s0 + shift, plane, fb, pol);
        } else {
          if (hview) {
            const int c0h = ch.rev ? s0 : s0 - pl.K;
            for (int q = 0; q < pl.nbh; ++q)
              tma_load3(dst + q * pl.bh * 32, &A.in[o][t], c0h, q * pl.bh, plane, fb, pol);
          } else {
            for (int q = 0; q < pl.nbh; ++q)
              tma_load3(dst + q * pl.bh * 16, &A.in[o][t], s0, q * pl.bh, plane, fb, pol);
          }
        }
      }
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
    }
  }
}

// Output tile store (issued by consumer thread 0 once the staging buffer is complete).
__device__ __forceinline__ void store_tile(const StreamArgs& A, const Chain& ch, int j, const uint8_t* buf, int nout,
                                           const int64_t* planes, uint64_t pol) {
  const Plan& pl = A.plan;
  const int o = ch.vert ? 0 : 1;
  const int s0 = tile_start(ch, j, pl.K);
  for (int t = 0; t < nout; ++t) {
    const uint32_t src = smem_u32(buf + static_cast<size_t>(t) * pl.tile_bytes);
    if (ch.vert) {
      for (int q = 0; q < pl.nbw; ++q)
        tma_store3(&A.out[o][t], src + q * pl.K * pl.bw * pl.es, q * pl.bw, s0, static_cast<int>(planes[t]), pol);
    } else {
      for (int q = 0; q < pl.nbh; ++q)
        tma_store3(&A.out[o][t], src + q * pl.bh * 16, s0, q * pl.bh, static_cast<int>(planes[t]), pol);
    }
  }
  bulk_commit();
}

// Cross-warp neighbour values of one step: every warp publishes the value at its first and last
// position; lane 0 receives the left neighbour's last, lane 31 the right neighbour's first.
// Double-buffered by step parity, so one named barrier per step suffices.
__device__ __forceinline__ void halo_xchg(float* halo, int& par, int wi, int nwc, int lane, float first, float last,
                                          float& from_left, float& from_right) {
  from_left = 0.f;
  from_right = 0.f;
  if (nwc > 1) {
    float* hb = halo + par * (2 * kHaloW);
    if (lane == 0) hb[wi] = first;
    if (lane == 31) hb[kHaloW + wi] = last;
    named_bar(kBarStep, nwc * 32);
    if (lane == 0 && wi > 0) from_left = hb[kHaloW + wi - 1];
    if (lane == 31 && wi < nwc - 1) from_right = hb[wi + 1];
    par ^= 1;
  }
}

__device__ __forceinline__ float shfl_idx(float v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// ------------------------------------------------------------------------------ forward consumer

// Vertical tile: up to K steps; lane owns positions r0, r0+1.
template <typename T>
__device__ __forceinline__ void fwd_tile_vert(const Plan& pl, const TileGeom& tg, const Chain& ch, int j,
                                              const uint8_t* st, uint8_t* ob, float* halo, int& par, int wi, int lane,
                                              float (&h)[2], bool prenorm) {
  const int r0 = wi * kLanePos + lane * kE;
  bool valid[2], hl[2], hr[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    valid[e] = (r0 + e) < ch.P;
    hl[e] = (r0 + e) >= 1;
    hr[e] = (r0 + e) <= ch.P - 2;
  }
  for (int tt = 0; tt < pl.K; ++tt) {
    const int t = j * pl.K + tt;
    if (t >= ch.L) break;
    const int kk = ch.rev ? (pl.K - 1 - tt) : tt;
    const uint32_t off = tg.vert(kk, r0);
    float x[2], lam[2], wl[2], wm[2], wr[2];
    V2<T>::load(st + F_X * pl.tile_bytes + off, x);
    V2<T>::load(st + F_LAM * pl.tile_bytes + off, lam);
    V2<T>::load(st + F_WL * pl.tile_bytes + off, wl);
    V2<T>::load(st + F_WM * pl.tile_bytes + off, wm);
    V2<T>::load(st + F_WR * pl.tile_bytes + off, wr);
    float left = shfl_idx(h[1], (lane + 31) & 31);
    float right = shfl_idx(h[0], (lane + 1) & 31);
    float fl, fr;
    halo_xchg(halo, par, wi, pl.nwc, lane, h[0], h[1], fl, fr);
    if (lane == 0) left = fl;
    if (lane == 31) right = fr;
    float hn[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float l = hl[e] ? wl[e] : 0.f;
      const float r = hr[e] ? wr[e] : 0.f;
      const float hm1 = (e == 0) ? left : h[0];
      const float hp1 = (e == 1) ? right : h[1];
      const float acc = fmaf(l, hm1, fmaf(wm[e], h[e], r * hp1));
      const float inv = prenorm ? 1.f : fast_rcp(wm[e] + l + r);
      hn[e] = valid[e] ? fmaf(acc, inv, lam[e] * x[e]) : 0.f;
    }
    h[0] = hn[0];
    h[1] = hn[1];
    V2<T>::store(ob + off, h);
  }
}

// Horizontal tile: K steps (one 16-byte row chunk per tensor); lane owns rows wi*64 + q*32 + lane.
template <typename T, bool kRev>
__device__ __forceinline__ void fwd_tile_horiz(const Plan& pl, const Chain& ch, int j, const uint8_t* st, uint8_t* ob,
                                               float* halo, int& par, int wi, int lane, float (&h)[2], bool prenorm) {
  constexpr int K = Row<T>::K;
  uint4 X[kNS], LAM[kNS], WL[kNS], WM[kNS], WR[kNS], OUT[kNS];
  bool valid[kNS], hl[kNS], hr[kNS];
#pragma unroll
  for (int q = 0; q < kNS; ++q) {
    const int r = wi * kLanePos + q * 32 + lane;
    valid[q] = r < ch.P;
    hl[q] = r >= 1;
    hr[q] = r <= ch.P - 2;
    const uint32_t off = static_cast<uint32_t>(r * 16);
    X[q] = *reinterpret_cast<const uint4*>(st + F_X * pl.tile_bytes + off);
    LAM[q] = *reinterpret_cast<const uint4*>(st + F_LAM * pl.tile_bytes + off);
    WL[q] = *reinterpret_cast<const uint4*>(st + F_WL * pl.tile_bytes + off);
    WM[q] = *reinterpret_cast<const uint4*>(st + F_WM * pl.tile_bytes + off);
    WR[q] = *reinterpret_cast<const uint4*>(st + F_WR * pl.tile_bytes + off);
    OUT[q] = make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int tt = 0; tt < K; ++tt) {
    const int t = j * K + tt;
    if (t < ch.L) {
      const int kk = kRev ? (K - 1 - tt) : tt;
      float up[kNS], dn[kNS];
#pragma unroll
      for (int q = 0; q < kNS; ++q) {
        up[q] = shfl_idx(h[q], (lane + 31) & 31);
        dn[q] = shfl_idx(h[q], (lane + 1) & 31);
      }
      float fl, fr;
      halo_xchg(halo, par, wi, pl.nwc, lane, h[0], h[kNS - 1], fl, fr);
      float hn[kNS];
#pragma unroll
      for (int q = 0; q < kNS; ++q) {
        const float hm1 = (lane == 0) ? (q == 0 ? fl : up[q > 0 ? q - 1 : 0]) : up[q];
        const float hp1 = (lane == 31) ? (q == kNS - 1 ? fr : dn[q + 1 < kNS ? q + 1 : q]) : dn[q];
        const float wlv = hl[q] ? Row<T>::get(WL[q], kk) : 0.f;
        const float wrv = hr[q] ? Row<T>::get(WR[q], kk) : 0.f;
        const float wmv = Row<T>::get(WM[q], kk);
        const float acc = fmaf(wlv, hm1, fmaf(wmv, h[q], wrv * hp1));
        const float inv = prenorm ? 1.f : fast_rcp(wmv + wlv + wrv);
        hn[q] = valid[q] ? fmaf(acc, inv, Row<T>::get(LAM[q], kk) * Row<T>::get(X[q], kk)) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < kNS; ++q) {
        h[q] = hn[q];
        Row<T>::set(OUT[q], kk, hn[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kNS; ++q) {
    const int r = wi * kLanePos + q * 32 + lane;
    *reinterpret_cast<uint4*>(ob + r * 16) = OUT[q];
  }
}

template <typename T, int kMaxNWC>
__global__ void __launch_bounds__((kMaxNWC + 1) * 32, 1) fwd_stream_kernel(const __grid_constant__ StreamArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  const Plan& pl = A.plan;
  uint8_t* ring = smem;
  uint8_t* outbuf = ring + static_cast<size_t>(pl.nstages) * pl.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(outbuf + 2 * static_cast<size_t>(pl.out_bytes));
  uint64_t* empty = full + pl.nstages;
  float* halo = reinterpret_cast<float*>(empty + pl.nstages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < pl.nstages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), pl.nwc);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == pl.nwc) {  // producer warp
    if (lane == 0) {
      for (int o = 0; o < 2; ++o)
        for (int t = 0; t < F_NIN; ++t) asm volatile("prefetch.tensormap [%0];" ::"l"(&A.in[o][t]) : "memory");
      producer_loop<false>(A, ring, full, empty);
    }
    return;
  }
  const bool prenorm = A.p.flags & GSPN_FLAG_PRENORMALIZED;
  const uint64_t pol_out = policy_evict_first();
  TileGeom tg;
  tg.K = pl.K;
  tg.bw_log2 = 31 - __clz(pl.bw);
  tg.es = pl.es;
  const int nthreads = pl.nwc * 32;
  int stage = 0, par = 0, ob_sel = 0;
  uint32_t phase = 0;
  for (int64_t w = blockIdx.x; w < pl.nchains; w += gridDim.x) {
    const Chain ch = make_chain(A.p, pl.K, w);
    float h[2] = {0.f, 0.f};
    for (int j = 0; j < ch.ntiles; ++j) {
      mbar_wait(smem_u32(&full[stage]), phase);
      const uint8_t* st = ring + static_cast<size_t>(stage) * pl.stage_bytes;
      uint8_t* ob = outbuf + static_cast<size_t>(ob_sel) * pl.out_bytes;
      if (ch.vert) {
        fwd_tile_vert<T>(pl, tg, ch, j, st, ob, halo, par, warp, lane, h, prenorm);
      } else if (ch.rev) {
        fwd_tile_horiz<T, true>(pl, ch, j, st, ob, halo, par, warp, lane, h, prenorm);
      } else {
        fwd_tile_horiz<T, false>(pl, ch, j, st, ob, halo, par, warp, lane, h, prenorm);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[stage]));
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
      fence_proxy_async();
      named_bar(kBarTile, nthreads);
      if (threadIdx.x == 0) {
        const int64_t planes[1] = {ch.chain};
        store_tile(A, ch, j, ob, 1, planes, pol_out);
        bulk_wait_read1();
      }
      named_bar(kBarTile, nthreads);
      ob_sel ^= 1;
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// ------------------------------------------------------------------------------ backward consumer

// Vertical backward tile (reverse step order). ea/eb/ec carry a_{t+1} g_{t+1}, b_{t+1} g_{t+1},
// c_{t+1} g_{t+1} of this lane's positions from the previously processed step.
template <typename T, bool kGrouped>
__device__ __forceinline__ void bwd_tile_vert(const StreamArgs& A, const TileGeom& tg, const Chain& ch, int j,
                                              const uint8_t* st, uint8_t* ob, float* halo, int& par, int wi,
                                              int lane, float (&ea)[2], float (&eb)[2], float (&ec)[2], bool prenorm,
                                              uint64_t pol_acc) {
  const Plan& pl = A.plan;
  const ScanParams& p = A.p;
  const int r0 = wi * kLanePos + lane * kE;
  bool valid[2], hl[2], hr[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    valid[e] = (r0 + e) < ch.P;
    hl[e] = (r0 + e) >= 1;
    hr[e] = (r0 + e) <= ch.P - 2;
  }
  const int64_t HW = p.H * p.W;
  float* dxacc = p.dx_acc + ch.bc * HW;
  float* dwa_l = kGrouped ? p.dwa_l + ch.wplane * HW : nullptr;
  float* dwa_m = kGrouped ? p.dwa_m + ch.wplane * HW : nullptr;
  float* dwa_r = kGrouped ? p.dwa_r + ch.wplane * HW : nullptr;
  const int rl = (r0 >= 1) ? r0 - 1 : 0;  // clamped neighbour positions (masked by hl/hr)
  const int rr = (r0 + 2 < pl.ppad) ? r0 + 2 : r0 + 1;
  for (int tt = pl.K - 1; tt >= 0; --tt) {
    const int t = j * pl.K + tt;
    if (t >= ch.L) continue;
    const int kk = ch.rev ? (pl.K - 1 - tt) : tt;
    const uint32_t off = tg.vert(kk, r0);
    float x[2], lam[2], dh[2], wl[2], wm[2], wr[2], hp[2];
    V2<T>::load(st + B_X * pl.tile_bytes + off, x);
    V2<T>::load(st + B_LAM * pl.tile_bytes + off, lam);
    V2<T>::load(st + B_DH * pl.tile_bytes + off, dh);
    V2<T>::load(st + B_WL * pl.tile_bytes + off, wl);
    V2<T>::load(st + B_WM * pl.tile_bytes + off, wm);
    V2<T>::load(st + B_WR * pl.tile_bytes + off, wr);
    V2<T>::load(st + B_H * pl.tile_bytes + off, hp);
    const uint8_t* hb = st + B_H * pl.tile_bytes;
    const float hpl = to_f(*reinterpret_cast<const T*>(hb + tg.vert(kk, rl)));
    const float hpr = to_f(*reinterpret_cast<const T*>(hb + tg.vert(kk, rr)));
    // g_t = dh_t + b_{t+1} g_{t+1} + a_{t+1}[r+1] g_{t+1}[r+1] + c_{t+1}[r-1] g_{t+1}[r-1]
    float from_right = shfl_idx(ea[0], (lane + 1) & 31);  // a g of position r0+2
    float from_left = shfl_idx(ec[1], (lane + 31) & 31);  // c g of position r0-1
    float fl, fr;
    halo_xchg(halo, par, wi, pl.nwc, lane, ea[0], ec[1], fl, fr);
    if (lane == 0) from_left = fl;
    if (lane == 31) from_right = fr;
    float g[2];
    g[0] = valid[0] ? (dh[0] + eb[0] + ea[1] + from_left) : 0.f;
    g[1] = valid[1] ? (dh[1] + eb[1] + from_right + ec[0]) : 0.f;
    float dlam[2], dwl[2], dwm[2], dwr[2], Da[2], Db[2], Dc[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float l = hl[e] ? wl[e] : 0.f;
      const float r = hr[e] ? wr[e] : 0.f;
      const float inv = prenorm ? 1.f : fast_rcp(wm[e] + l + r);
      const float a = l * inv, b = wm[e] * inv, c = r * inv;
      dlam[e] = g[e] * x[e];
      const float hm1 = (e == 0) ? hpl : hp[0];
      const float hp1 = (e == 1) ? hpr : hp[1];
      Da[e] = hl[e] ? g[e] * hm1 : 0.f;
      Db[e] = g[e] * hp[e];
      Dc[e] = hr[e] ? g[e] * hp1 : 0.f;
      if (!kGrouped) {
        if (prenorm) {
          dwl[e] = Da[e]; dwm[e] = Db[e]; dwr[e] = Dc[e];
        } else {  // normalisation Jacobian (gspn_common.cuh: jacobian), inv = 1/S
          const float inv2 = inv * inv;
          dwl[e] = hl[e] ? fmaf(wm[e] + r, Da[e], -fmaf(wm[e], Db[e], r * Dc[e])) * inv2 : 0.f;
          dwm[e] = valid[e] ? fmaf(l + r, Db[e], -fmaf(l, Da[e], r * Dc[e])) * inv2 : 0.f;
          dwr[e] = hr[e] ? fmaf(l + wm[e], Dc[e], -fmaf(l, Da[e], wm[e] * Db[e])) * inv2 : 0.f;
        }
      }
      ea[e] = valid[e] ? a * g[e] : 0.f;
      eb[e] = valid[e] ? b * g[e] : 0.f;
      ec[e] = valid[e] ? c * g[e] : 0.f;
    }
    V2<T>::store(ob + O_DLAM * pl.tile_bytes + off, dlam);
    if (!kGrouped) {
      V2<T>::store(ob + O_DWL * pl.tile_bytes + off, dwl);
      V2<T>::store(ob + O_DWM * pl.tile_bytes + off, dwm);
      V2<T>::store(ob + O_DWR * pl.tile_bytes + off, dwr);
    }
    if (valid[0]) {  // W % 2 == 0 on this path: both positions valid or both padding
      const int row = ch.rev ? (ch.L - 1 - t) : t;
      const int64_t o = static_cast<int64_t>(row) * p.W + r0;
      red_add_v2(dxacc + o, g[0] * lam[0], g[1] * lam[1], pol_acc);
      if (kGrouped && t >= 1) {
        red_add_v2(dwa_l + o, Da[0], Da[1], pol_acc);
        red_add_v2(dwa_m + o, Db[0], Db[1], pol_acc);
        red_add_v2(dwa_r + o, Dc[0], Dc[1], pol_acc);
      }
    }
  }
}

// Horizontal backward tile (reverse step order); lane owns rows wi*64 + q*32 + lane.
template <typename T, bool kRev, bool kGrouped>
__device__ __forceinline__ void bwd_tile_horiz(const StreamArgs& A, const Chain& ch, int j, const uint8_t* st,
                                               uint8_t* ob, float* halo, int& par, int wi, int lane, float (&ea)[2],
                                               float (&eb)[2], float (&ec)[2], bool prenorm, uint64_t pol_acc) {
  constexpr int K = Row<T>::K;
  constexpr int es = static_cast<int>(sizeof(T));
  const Plan& pl = A.plan;
  const ScanParams& p = A.p;
  const int64_t HW = p.H * p.W;
  float* dxacc = p.dx_acc + ch.bc * HW;
  float* dwa_l = kGrouped ? p.dwa_l + ch.wplane * HW : nullptr;
  float* dwa_m = kGrouped ? p.dwa_m + ch.wplane * HW : nullptr;
  float* dwa_r = kGrouped ? p.dwa_r + ch.wplane * HW : nullptr;
  const int c0 = tile_start(ch, j, K);  // canonical column of kk = 0 (W % K == 0 on this path)
  bool valid[kNS], hl[kNS], hr[kNS];
  uint4 X[kNS], LAM[kNS], DH[kNS], WL[kNS], WM[kNS], WR[kNS], HP0[kNS], HP1[kNS];
  // h tile: rows of 2K steps (32 bytes) with the TMA 32-byte swizzle (16-byte chunk ^= row bit 2)
  const uint8_t* hbase = st + B_H * pl.tile_bytes;
  auto swz = [](int r, int c) { return static_cast<uint32_t>(r * 32 + ((c ^ ((r >> 2) & 1)) << 4)); };
  uint4 O0[kNS], O1[kNS], O2[kNS], O3[kNS];
  float DX[kNS][K];
#pragma unroll
  for (int q = 0; q < kNS; ++q) {
    const int r = wi * kLanePos + q * 32 + lane;
    valid[q] = r < ch.P;
    hl[q] = r >= 1;
    hr[q] = r <= ch.P - 2;
    const uint32_t off = static_cast<uint32_t>(r * 16);
    X[q] = *reinterpret_cast<const uint4*>(st + B_X * pl.tile_bytes + off);
    LAM[q] = *reinterpret_cast<const uint4*>(st + B_LAM * pl.tile_bytes + off);
    DH[q] = *reinterpret_cast<const uint4*>(st + B_DH * pl.tile_bytes + off);
    WL[q] = *reinterpret_cast<const uint4*>(st + B_WL * pl.tile_bytes + off);
    WM[q] = *reinterpret_cast<const uint4*>(st + B_WM * pl.tile_bytes + off);
    WR[q] = *reinterpret_cast<const uint4*>(st + B_WR * pl.tile_bytes + off);
    HP0[q] = *reinterpret_cast<const uint4*>(hbase + swz(r, 0));
    HP1[q] = *reinterpret_cast<const uint4*>(hbase + swz(r, 1));
    O0[q] = O1[q] = O2[q] = O3[q] = make_uint4(0, 0, 0, 0);
  }
  // rows just outside this warp's range (for h_{t-1}[r-1] of lane 0 / [r+1] of lane 31)
  const int row_lo = wi * kLanePos - 1, row_hi = wi * kLanePos + kLanePos;
  const int rlo = row_lo >= 0 ? row_lo : 0;
  const int rhi = row_hi < pl.ppad ? row_hi : pl.ppad - 1;
#pragma unroll
  for (int tt = K - 1; tt >= 0; --tt) {
    const int t = j * K + tt;
    const int kk = kRev ? (K - 1 - tt) : tt;
    const int he = kRev ? (kk + 1) : (K + kk - 1);  // h_{t-1} element in the 2K-step h row
    if (t < ch.L) {
      float from_right[kNS], from_left[kNS], hv[kNS], hup[kNS], hdn[kNS];
#pragma unroll
      for (int q = 0; q < kNS; ++q) {
        from_right[q] = shfl_idx(ea[q], (lane + 1) & 31);
        from_left[q] = shfl_idx(ec[q], (lane + 31) & 31);
        hv[q] = (he < K) ? Row<T>::get(HP0[q], he) : Row<T>::get(HP1[q], he - K);
        hup[q] = shfl_idx(hv[q], (lane + 31) & 31);
        hdn[q] = shfl_idx(hv[q], (lane + 1) & 31);
      }
      const float h_lo = to_f(*reinterpret_cast<const T*>(hbase + swz(rlo, he / K) + (he % K) * es));
      const float h_hi = to_f(*reinterpret_cast<const T*>(hbase + swz(rhi, he / K) + (he % K) * es));
      float fl, fr;
      halo_xchg(halo, par, wi, pl.nwc, lane, ea[0], ec[kNS - 1], fl, fr);
#pragma unroll
      for (int q = 0; q < kNS; ++q) {
        const float nr = (lane == 31) ? (q == kNS - 1 ? fr : from_right[q + 1 < kNS ? q + 1 : q]) : from_right[q];
        const float nl = (lane == 0) ? (q == 0 ? fl : from_left[q > 0 ? q - 1 : 0]) : from_left[q];
        const float hpl = (lane == 0) ? (q == 0 ? h_lo : hup[q > 0 ? q - 1 : 0]) : hup[q];
        const float hpr = (lane == 31) ? (q == kNS - 1 ? h_hi : hdn[q + 1 < kNS ? q + 1 : q]) : hdn[q];
        const float g = valid[q] ? (Row<T>::get(DH[q], kk) + eb[q] + nr + nl) : 0.f;
        const float wl = Row<T>::get(WL[q], kk), wm = Row<T>::get(WM[q], kk), wr = Row<T>::get(WR[q], kk);
        const float l = hl[q] ? wl : 0.f;
        const float rr = hr[q] ? wr : 0.f;
        const float inv = prenorm ? 1.f : fast_rcp(wm + l + rr);
        const float a = l * inv, b = wm * inv, c = rr * inv;
        const float Da = hl[q] ? g * hpl : 0.f;
        const float Db = g * hv[q];
        const float Dc = hr[q] ? g * hpr : 0.f;
        Row<T>::set(O0[q], kk, g * Row<T>::get(X[q], kk));
        if (!kGrouped) {
          float dwl, dwm, dwr;
          if (prenorm) {
            dwl = Da; dwm = Db; dwr = Dc;
          } else {  // normalisation Jacobian (gspn_common.cuh: jacobian), inv = 1/S
            const float inv2 = inv * inv;
            dwl = hl[q] ? fmaf(wm + rr, Da, -fmaf(wm, Db, rr * Dc)) * inv2 : 0.f;
            dwm = valid[q] ? fmaf(l + rr, Db, -fmaf(l, Da, rr * Dc)) * inv2 : 0.f;
            dwr = hr[q] ? fmaf(l + wm, Dc, -fmaf(l, Da, wm * Db)) * inv2 : 0.f;
          }
          Row<T>::set(O1[q], kk, dwl);
          Row<T>::set(O2[q], kk, dwm);
          Row<T>::set(O3[q], kk, dwr);
        } else if (valid[q] && t >= 1) {
          const int r = wi * kLanePos + q * 32 + lane;
          const int64_t o = static_cast<int64_t>(r) * p.W + c0 + kk;
          red_add_f32(dwa_l + o, Da, pol_acc);
          red_add_f32(dwa_m + o, Db, pol_acc);
          red_add_f32(dwa_r + o, Dc, pol_acc);
        }
        DX[q][kk] = g * Row<T>::get(LAM[q], kk);
        ea[q] = valid[q] ? a * g : 0.f;
        eb[q] = valid[q] ? b * g : 0.f;
        ec[q] = valid[q] ? c * g : 0.f;
      }
    } else {
#pragma unroll
      for (int q = 0; q < kNS; ++q) DX[q][kk] = 0.f;
    }
  }
#pragma unroll
  for (int q = 0; q < kNS; ++q) {
    const int r = wi * kLanePos + q * 32 + lane;
    *reinterpret_cast<uint4*>(ob + O_DLAM * pl.tile_bytes + r * 16) = O0[q];
    if (!kGrouped) {
      *reinterpret_cast<uint4*>(ob + O_DWL * pl.tile_bytes + r * 16) = O1[q];
      *reinterpret_cast<uint4*>(ob + O_DWM * pl.tile_bytes + r * 16) = O2[q];
      *reinterpret_cast<uint4*>(ob + O_DWR * pl.tile_bytes + r * 16) = O3[q];
    }
    if (valid[q]) {
      const int64_t o = static_cast<int64_t>(r) * p.W + c0;
#pragma unroll
      for (int v = 0; v < K; v += 4) red_add_v4(dxacc + o + v, DX[q][v], DX[q][v + 1], DX[q][v + 2], DX[q][v + 3], pol_acc);
    }
  }
}

// The last of a plane's D chains converts the fp32 dx accumulator; the last of a group's C/G channels
// applies the normalisation Jacobian to the group-summed tap gradients:
// q = a Da + b Db + c Dc; dw_l = [r>=1](Da - q)/S, dw_m = (Db - q)/S, dw_r = [r<=P-2](Dc - q)/S.
template <typename T, bool kGrouped>
__device__ void bwd_chain_epilogue(const StreamArgs& A, const Chain& ch, int* flag, int nthreads) {
  const ScanParams& p = A.p;
  const int64_t HW = p.H * p.W;
  __threadfence();
  named_bar(kBarTile, nthreads);
  if (threadIdx.x == 0) {
    int f = 0;
    if (atomicAdd(&p.counters[ch.bc], 1u) == static_cast<unsigned>(p.D - 1)) f |= 1;
    if (kGrouped && atomicAdd(&p.counters[p.B * p.C + ch.wplane], 1u) == static_cast<unsigned>(p.C / p.G - 1))
      f |= 2;
    *flag = f;
  }
  named_bar(kBarTile, nthreads);
  const int f = *flag;
  named_bar(kBarTile, nthreads);  // flag slot reusable by the next chain
  if (f) __threadfence();
  if (f & 1) {
    const float4* src = reinterpret_cast<const float4*>(p.dx_acc + ch.bc * HW);
    T* dst = static_cast<T*>(p.dx) + ch.bc * HW;
    for (int64_t i = threadIdx.x; i < HW / 4; i += nthreads) store4<T>(dst + 4 * i, __ldcg(src + i));
  }
  if (kGrouped && (f & 2)) {
    const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
    const int64_t base = ch.wplane * HW;
    const bool vert = ch.vert;
    const int64_t P = vert ? p.W : p.H;
    for (int64_t i = threadIdx.x; i < HW; i += nthreads) {
      const int64_t r = vert ? (i % p.W) : (i / p.W);
      const bool hl = r >= 1, hr = r <= P - 2;
      const float Da = __ldcg(p.dwa_l + base + i), Db = __ldcg(p.dwa_m + base + i), Dc = __ldcg(p.dwa_r + base + i);
      const float wl = to_f(static_cast<const T*>(p.wl)[base + i]);
      const float wm = to_f(static_cast<const T*>(p.wm)[base + i]);
      const float wr = to_f(static_cast<const T*>(p.wr)[base + i]);
      float ol, om, orr;
      jacobian(wl, wm, wr, hl, hr, prenorm, Da, Db, Dc, ol, om, orr);
      static_cast<T*>(p.dwl)[base + i] = from_f<T>(ol);
      static_cast<T*>(p.dwm)[base + i] = from_f<T>(om);
      static_cast<T*>(p.dwr)[base + i] = from_f<T>(orr);
    }
  }
}

template <typename T, bool kGrouped, int kMaxNWC>
__global__ void __launch_bounds__((kMaxNWC + 1) * 32, 1) bwd_stream_kernel(const __grid_constant__ StreamArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared address space
  const Plan& pl = A.plan;
  uint8_t* ring = smem;
  uint8_t* outbuf = ring + static_cast<size_t>(pl.nstages) * pl.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(outbuf + 2 * static_cast<size_t>(pl.out_bytes));
  uint64_t* empty = full + pl.nstages;
  float* halo = reinterpret_cast<float*>(empty + pl.nstages);
  int* flag = reinterpret_cast<int*>(halo + 4 * kHaloW);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < pl.nstages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), pl.nwc);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == pl.nwc) {
    if (lane == 0) {
      for (int o = 0; o < 2; ++o)
        for (int t = 0; t < B_NIN; ++t) asm volatile("prefetch.tensormap [%0];" ::"l"(&A.in[o][t]) : "memory");
      producer_loop<true>(A, ring, full, empty);
    }
    return;
  }
  const bool prenorm = A.p.flags & GSPN_FLAG_PRENORMALIZED;
  const uint64_t pol_out = policy_evict_first();
  const uint64_t pol_acc = policy_evict_last();
  TileGeom tg;
  tg.K = pl.K;
  tg.bw_log2 = 31 - __clz(pl.bw);
  tg.es = pl.es;
  const int nthreads = pl.nwc * 32;
  int stage = 0, par = 0, ob_sel = 0;
  uint32_t phase = 0;
  for (int64_t w = blockIdx.x; w < pl.nchains; w += gridDim.x) {
    const Chain ch = make_chain(A.p, pl.K, w);
    float ea[2] = {0.f, 0.f}, eb[2] = {0.f, 0.f}, ec[2] = {0.f, 0.f};
    for (int jj = 0; jj < ch.ntiles; ++jj) {
      const int j = ch.ntiles - 1 - jj;
      mbar_wait(smem_u32(&full[stage]), phase);
      const uint8_t* st = ring + static_cast<size_t>(stage) * pl.stage_bytes;
      uint8_t* ob = outbuf + static_cast<size_t>(ob_sel) * pl.out_bytes;
      if (ch.vert) {
        bwd_tile_vert<T, kGrouped>(A, tg, ch, j, st, ob, halo, par, warp, lane, ea, eb, ec, prenorm, pol_acc);
      } else if (ch.rev) {
        bwd_tile_horiz<T, true, kGrouped>(A, ch, j, st, ob, halo, par, warp, lane, ea, eb, ec, prenorm, pol_acc);
      } else {
        bwd_tile_horiz<T, false, kGrouped>(A, ch, j, st, ob, halo, par, warp, lane, ea, eb, ec, prenorm, pol_acc);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[stage]));
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
      fence_proxy_async();
      named_bar(kBarTile, nthreads);
      if (threadIdx.x == 0) {
        const int64_t planes[4] = {ch.chain, ch.wplane, ch.wplane, ch.wplane};
        store_tile(A, ch, j, ob, kGrouped ? 1 : 4, planes, pol_out);
        bulk_wait_read1();
      }
      named_bar(kBarTile, nthreads);
      ob_sel ^= 1;
    }
    bwd_chain_epilogue<T, kGrouped>(A, ch, flag, nthreads);
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// ------------------------------------------------------------------------------------- host side

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

bool encode(CUtensorMap* m, const void* base, gspn_dtype_t dt, int64_t W, int64_t H, int64_t planes, int box0,
            int box1, bool promote, bool swizzle32 = false) {
  auto fn = get_encode();
  if (!fn) return false;
  const size_t s = dt == GSPN_BF16 ? 2 : 4;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(planes)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(W * s), static_cast<cuuint64_t>(W * H * s)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box0), static_cast<cuuint32_t>(box1), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, dt == GSPN_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  promote ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int smem_optin() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (n <= 0) n = 227 * 1024;
  }
  return n;
}

// Largest power-of-two box extent (<= 256, >= min_box) whose boxes tile n positions inside ppad.
int pick_box(int64_t n, int ppad, int min_box) {
  for (int b = 256; b >= min_box; b >>= 1)
    if (((n + b - 1) / b) * b <= ppad) return b;
  return 0;
}

// Shape eligibility + plan. nin/nout: tensors per tile.
bool make_plan(const ScanParams& p, gspn_dtype_t dt, int nin, int nout, int min_stages, Plan* pl) {
  const int s = dt == GSPN_BF16 ? 2 : 4;
  if ((p.W * s) % 16 != 0) return false;  // TMA global stride alignment; also K | W for horizontal tiles
  bool any_v = false, any_h = false;
  for (int k = 0; k < p.D; ++k) {
    if (p.dirbit[k] == GSPN_DIR_T2B || p.dirbit[k] == GSPN_DIR_B2T) any_v = true; else any_h = true;
  }
  const int64_t maxP = std::max<int64_t>(any_v ? p.W : 0, any_h ? p.H : 0);
  if (maxP > static_cast<int64_t>(kLanePos) * kHaloW) return false;
  memset(pl, 0, sizeof *pl);
  pl->K = 16 / s;
  pl->es = s;
  pl->nwc = static_cast<int>((maxP + kLanePos - 1) / kLanePos);
  pl->ppad = kLanePos * pl->nwc;
  pl->bw = pick_box(p.W, pl->ppad, 16 / s);
  pl->bh = pick_box(p.H, pl->ppad, 1);
  if (any_v && pl->bw == 0) return false;
  if (any_h && pl->bh == 0) return false;
  if (pl->bw == 0) pl->bw = 16 / s;
  if (pl->bh == 0) pl->bh = 1;
  pl->nbw = static_cast<int>((p.W + pl->bw - 1) / pl->bw);
  pl->nbh = static_cast<int>((p.H + pl->bh - 1) / pl->bh);
  pl->nin = nin;
  pl->nout = nout;
  pl->tile_bytes = static_cast<uint32_t>(pl->K * pl->ppad * s);
  pl->h_wide = (nin == B_NIN) ? 1 : 0;
  pl->stage_bytes = (nin + pl->h_wide) * pl->tile_bytes;
  pl->out_bytes = nout * pl->tile_bytes;
  pl->tx_v = static_cast<uint32_t>(nin * pl->nbw * pl->bw * pl->K * s);
  pl->tx_h = static_cast<uint32_t>((nin + pl->h_wide) * pl->nbh * pl->bh * pl->K * s);
  const int budget = smem_optin() - 1024 /*alignment*/ - 512 /*barriers, halo, flag*/;
  const int avail = budget - 2 * static_cast<int>(pl->out_bytes);
  int ns = avail / static_cast<int>(pl->stage_bytes);
  if (ns > 8) ns = 8;
  if (ns < min_stages) return false;
  pl->nstages = ns;
  pl->nchains = p.D * p.B * p.C;
  pl->smem_bytes = 1024 + ns * pl->stage_bytes + 2 * pl->out_bytes + 512;
  return true;
}

bool fill_maps(StreamArgs* A, const void* const* ins, int nin, void* const* outs, const int64_t* in_planes,
               const int64_t* out_planes, int nout, gspn_dtype_t dt) {
  const Plan& pl = A->plan;
  const ScanParams& p = A->p;
  for (int t = 0; t < nin; ++t) {
    if (!encode(&A->in[0][t], ins[t], dt, p.W, p.H, in_planes[t], pl.bw, pl.K, false)) return false;
    const bool wide = pl.h_wide && t == nin - 1;  // bwd h_{t-1} view: 2K-step rows, 32-byte swizzle
    if (!encode(&A->in[1][t], ins[t], dt, p.W, p.H, in_planes[t], wide ? 2 * pl.K : pl.K, pl.bh, true, wide))
      return false;
  }
  for (int t = 0; t < nout; ++t) {
    if (!encode(&A->out[0][t], outs[t], dt, p.W, p.H, out_planes[t], pl.bw, pl.K, false)) return false;
    if (!encode(&A->out[1][t], outs[t], dt, p.W, p.H, out_planes[t], pl.K, pl.bh, false)) return false;
  }
  return true;
}

template <typename KernelT>
cudaError_t launch(KernelT kernel, const StreamArgs& A, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(A.plan.smem_bytes));
  if (e != cudaSuccess) return e;
  const int threads = (A.plan.nwc + 1) * 32;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, A.plan.smem_bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = static_cast<int64_t>(sm_count()) * per_sm;
  if (grid > A.plan.nchains) grid = A.plan.nchains;
  kernel<<<static_cast<unsigned>(grid), threads, A.plan.smem_bytes, s>>>(A);
  return cudaGetLastError();
}

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

struct WsLayout {
  size_t dx, dwa, cnt, total, zero_bytes;
};

WsLayout ws_layout(int64_t B, int64_t C, int64_t H, int64_t W, int64_t D, int64_t G) {
  WsLayout l;
  l.dx = 0;
  size_t off = align_up(static_cast<size_t>(B * C * H * W) * sizeof(float));
  l.dwa = off;
  if (G < C) off += 3 * align_up(static_cast<size_t>(D * B * G * H * W) * sizeof(float));
  l.cnt = off;
  off += align_up(static_cast<size_t>(B * C + D * B * G) * sizeof(unsigned));
  l.total = off;
  l.zero_bytes = off;
  return l;
}

}  // namespace

size_t stream_bwd_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W, int64_t D, int64_t G, gspn_dtype_t) {
  return ws_layout(B, C, H, W, D, G).total;
}

cudaError_t launch_fwd_stream(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches, bool* handled) {
  *handled = false;
  static StreamArgs A;  // large (3 KB): keep off the stack; launches copy it into the parameter buffer
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  memset(&A, 0, sizeof A);
  A.p = p;
  if (!make_plan(p, dt, F_NIN, 1, 2, &A.plan)) return cudaSuccess;
  const void* ins[F_NIN] = {p.x, p.lam, p.wl, p.wm, p.wr};
  const int64_t in_planes[F_NIN] = {p.B * p.C, p.D * p.B * p.C, p.D * p.B * p.G, p.D * p.B * p.G, p.D * p.B * p.G};
  void* outs[1] = {p.hout};
  const int64_t out_planes[1] = {p.D * p.B * p.C};
  if (!fill_maps(&A, ins, F_NIN, outs, in_planes, out_planes, 1, dt)) return cudaSuccess;
  *handled = true;
  cudaError_t e;
  if (A.plan.nwc <= 8)
    e = dt == GSPN_BF16 ? launch(fwd_stream_kernel<__nv_bfloat16, 8>, A, s) : launch(fwd_stream_kernel<float, 8>, A, s);
  else
    e = dt == GSPN_BF16 ? launch(fwd_stream_kernel<__nv_bfloat16, 16>, A, s) : launch(fwd_stream_kernel<float, 16>, A, s);
  *launches += 1;
  return e;
}

cudaError_t launch_bwd_stream(const ScanParams& p0, gspn_dtype_t dt, cudaStream_t s, int* launches, bool* handled) {
  *handled = false;
  static StreamArgs A;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  memset(&A, 0, sizeof A);
  A.p = p0;
  ScanParams& p = A.p;
  const bool grouped = p.G < p.C;
  const int nout = grouped ? 1 : 4;
  if (!make_plan(p, dt, B_NIN, nout, 2, &A.plan)) return cudaSuccess;
  const WsLayout l = ws_layout(p.B, p.C, p.H, p.W, p.D, p.G);
  if (p.ws == nullptr || p.ws_bytes < l.total) return cudaSuccess;
  char* ws = static_cast<char*>(p.ws);
  p.dx_acc = reinterpret_cast<float*>(ws + l.dx);
  if (grouped) {
    const size_t nwb = align_up(static_cast<size_t>(p.D * p.B * p.G * p.H * p.W) * sizeof(float));
    p.dwa_l = reinterpret_cast<float*>(ws + l.dwa);
    p.dwa_m = reinterpret_cast<float*>(ws + l.dwa + nwb);
    p.dwa_r = reinterpret_cast<float*>(ws + l.dwa + 2 * nwb);
  }
  p.counters = reinterpret_cast<unsigned*>(ws + l.cnt);
  const void* ins[B_NIN] = {p.x, p.lam, p.dh, p.wl, p.wm, p.wr, p.h};
  const int64_t nbc = p.B * p.C, nc = p.D * p.B * p.C, nw = p.D * p.B * p.G;
  const int64_t in_planes[B_NIN] = {nbc, nc, nc, nw, nw, nw, nc};
  void* outs[4] = {p.dlam, p.dwl, p.dwm, p.dwr};
  const int64_t out_planes[4] = {nc, nw, nw, nw};
  if (!fill_maps(&A, ins, B_NIN, outs, in_planes, out_planes, nout, dt)) return cudaSuccess;
  *handled = true;
  cudaError_t e = cudaMemsetAsync(p.ws, 0, l.zero_bytes, s);
  if (e != cudaSuccess) return e;
  const bool small = A.plan.nwc <= 8;
  if (dt == GSPN_BF16) {
    if (small)
      e = grouped ? launch(bwd_stream_kernel<__nv_bfloat16, true, 8>, A, s) : launch(bwd_stream_kernel<__nv_bfloat16, false, 8>, A, s);
    else
      e = grouped ? launch(bwd_stream_kernel<__nv_bfloat16, true, 16>, A, s) : launch(bwd_stream_kernel<__nv_bfloat16, false, 16>, A, s);
  } else {
    if (small)
      e = grouped ? launch(bwd_stream_kernel<float, true, 8>, A, s) : launch(bwd_stream_kernel<float, false, 8>, A, s);
    else
      e = grouped ? launch(bwd_stream_kernel<float, true, 16>, A, s) : launch(bwd_stream_kernel<float, false, 16>, A, s);
  }
  *launches += 1;
  return e;
}

}  // namespace gspn
