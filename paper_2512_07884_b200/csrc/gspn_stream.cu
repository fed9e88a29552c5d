// gspn_stream.cu — the TMA-streaming fast path for sm_100a (B200).
//
// One persistent launch covers every requested direction ("Kernel Fuse"; the paper's
// one-stream-per-direction concurrency, becomes a direction dimension of the work queue).
// Work item = one chain (direction k, batch b, channel c): a P-wide state marching L steps. A CTA owns
// one chain at a time:
//  * warp NWC (the producer) streams K-step tiles (K * sizeof(T) = 16 bytes) of every input tensor
//    into a shared-memory ring with TMA (cp.async.bulk.tensor.3d, mbarrier complete_tx);
//  * NWC consumer warps run the recurrence with the carry in fp32 registers. A warp covers 128
//    consecutive positions: it OWNS the middle 128 - 2K and recomputes K "ghost" positions on each
//    side (temporal blocking): neighbours move by warp shuffles every step, and warps exchange their
//    edge values through shared memory once per K-step tile instead of once per step;
//  * outputs are staged in shared memory (double-buffered) and written back with TMA stores.
// Lane mappings (both conflict-free on the shared-memory tiles):
//   T2B/B2T (vertical):   tile = K image rows x P columns ([box][K][bw]); a lane owns 4 consecutive
//                         positions and reads one 4-element vector per tensor per step.
//   L2R/R2L (horizontal): tile = P image rows x 16 bytes ([P][K]); a lane owns 4 interleaved rows
//                         (position A + 32 q + lane) and holds the K steps of a row in one vector.
// Chains are ordered (b, c)-major with the D directions adjacent, so co-scheduled CTAs share a
// plane's x (and in the backward its fp32 dx accumulator) through L2.
//
// Backward: tiles in reverse step order; the carried state is
// (a g, b g, c g) of the previous step, so g_t = dh_t + (b g)[r] + (a g)[r+1] + (c g)[r-1];
// h_{t-1} comes from a second TMA view of h shifted one step against the scan (its zero fill at
// t = 0 is h_{-1} = 0); dx (sum over directions) accumulates with red.global.add into an fp32
// workspace plane that the last of the plane's D chains converts and discards from L2; per-channel
// dw gets the normalisation Jacobian in registers; grouped dw sums the normalised-tap gradients with
// red and the group's last channel applies the Jacobian.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "gspn_common.cuh"
#include "gspn_internal.h"

namespace gspn {
namespace {

constexpr int kMaxIn = 7;
constexpr int kMaxOut = 4;
constexpr int kEdgeW = 16;     // max consumer warps (edge-buffer slots)
constexpr int kBwdE2Warps = 12;  // consumer warps of the 2-positions-per-lane backward variant
constexpr int kBarTile = 1;    // named barrier ids (0 is __syncthreads): ghost exchange / epilogue
constexpr int kBarRows = 2;    // horizontal tiles: every warp holds its rows in registers

template <typename T>
struct Cfg {
  static constexpr int es = static_cast<int>(sizeof(T));
  static constexpr int K = 16 / es;             // steps per tile (one 16-byte row chunk)
  static constexpr int GH = K;                  // ghost positions on each side of a warp
  static constexpr int KS = 8 / es;             // bwd horizontal sub-tile (one 8-byte row chunk)
};

struct Plan {
  int K;               // steps per tile
  int own;             // owned positions per warp
  int nwc;             // consumer warps
  int ppad;            // positions held by a tile (>= P, multiple of 64 and of bw)
  int es;              // element size in bytes
  int bw, nbw;         // vertical TMA box width (positions) and box count
  int bh, nbh;         // horizontal TMA box height (positions) and box count
  int nin, nout;       // input / output tensors per tile
  int pair;            // load horizontal tiles in back-to-back pairs (ring of >= 3 stages)
  int null_compute;    // experiments only (GSPN_NULL=1): consumers skip the arithmetic (pipeline ceiling)
  int nosleep;         // experiments only (GSPN_NOSLEEP=1): producer polls instead of sleeping
  int h_wide;          // bwd: the last input (h) holds 2K steps for horizontal chains
  int nstages;
  uint32_t tile_bytes;   // one tensor's tile: K * ppad * es (= 16 * ppad)
  uint32_t stage_bytes;  // (nin + h_wide) * tile_bytes
  uint32_t tx_v, tx_h;   // TMA bytes landing per stage (vertical / horizontal chains)
  int64_t nchains;
  uint32_t smem_bytes;
  // L2 eviction priority per access class (0 evict_first, 1 evict_normal, 2 evict_last):
  // x loads, vertical loads, horizontal loads, vertical stores, horizontal stores, fp32 accumulators
  int pol[6];
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

// Wait with a suspend-time hint: the (single) producer thread sleeps in hardware instead of
// re-issuing try_wait, leaving its SMSP's issue slots to the consumer warps.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "WAITS%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITS%=;\n}" ::"r"(bar),
      "r"(parity), "r"(1000000u)
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
__device__ __forceinline__ uint64_t policy_evict_last();
__device__ __forceinline__ uint64_t policy_of(int code) {
  return code == 0 ? policy_evict_first() : (code == 1 ? policy_evict_normal() : policy_evict_last());
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


__device__ __forceinline__ void st_global_b32(void* p, uint32_t a, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(a), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_global_v2(void* p, uint32_t a, uint32_t b, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(a), "r"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_global_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

__device__ __forceinline__ float fast_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}


__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// Neighbour values inside a warp; the warp's outermost lanes get 0 (their positions are ghosts).
__device__ __forceinline__ float from_lower_lane(float v, int lane) {
  const float u = __shfl_up_sync(0xffffffffu, v, 1);
  return lane == 0 ? 0.f : u;
}
__device__ __forceinline__ float from_upper_lane(float v, int lane) {
  const float u = __shfl_down_sync(0xffffffffu, v, 1);
  return lane == 31 ? 0.f : u;
}

// ------------------------------------------------------------------------------ element access

// 4 consecutive elements of T in shared memory <-> floats (8 bytes for bf16, 16 for fp32).
template <typename T> struct V4;
template <> struct V4<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const uint8_t* p, float (&v)[4]) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    v[0] = __uint_as_float(u.x << 16); v[1] = __uint_as_float(u.x & 0xFFFF0000u);
    v[2] = __uint_as_float(u.y << 16); v[3] = __uint_as_float(u.y & 0xFFFF0000u);
  }
  static __device__ __forceinline__ uint2 pack(const float (&v)[4]) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
    __nv_bfloat162 b = __floats2bfloat162_rn(v[2], v[3]);
    return make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
  static __device__ __forceinline__ void store(uint8_t* p, const float (&v)[4]) {
    *reinterpret_cast<uint2*>(p) = pack(v);
  }
};
template <> struct V4<float> {
  static __device__ __forceinline__ void load(const uint8_t* p, float (&v)[4]) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
  }
  static __device__ __forceinline__ void store(uint8_t* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};

// 4 consecutive fp32 values -> T in global memory (dx conversion).
template <typename T> __device__ __forceinline__ void store4_global(T* p, float4 v);
template <> __device__ __forceinline__ void store4_global<__nv_bfloat16>(__nv_bfloat16* p, float4 v) {
  const float a[4] = {v.x, v.y, v.z, v.w};
  *reinterpret_cast<uint2*>(p) = V4<__nv_bfloat16>::pack(a);
}
template <> __device__ __forceinline__ void store4_global<float>(float* p, float4 v) {
  *reinterpret_cast<float4*>(p) = v;
}

// Element i of a packed row chunk (uint4 = 16 bytes, uint2 = 8 bytes) of T. i is a compile-time
// constant after unrolling, so the selects fold away.
template <typename T> struct Pk;
template <> struct Pk<__nv_bfloat16> {
  static __device__ __forceinline__ uint32_t word4(const uint4& u, int w) { return w == 0 ? u.x : w == 1 ? u.y : w == 2 ? u.z : u.w; }
  static __device__ __forceinline__ float get(const uint4& u, int i) {
    const uint32_t w = word4(u, i >> 1);
    return (i & 1) ? __uint_as_float(w & 0xFFFF0000u) : __uint_as_float(w << 16);
  }
  static __device__ __forceinline__ float get(const uint2& u, int i) {
    const uint32_t w = (i >> 1) ? u.y : u.x;
    return (i & 1) ? __uint_as_float(w & 0xFFFF0000u) : __uint_as_float(w << 16);
  }
  static __device__ __forceinline__ uint32_t bits(float v) {
    return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v)));
  }
  static __device__ __forceinline__ void set(uint4& u, int i, float v) {
    uint32_t& w = (i >> 1) == 0 ? u.x : (i >> 1) == 1 ? u.y : (i >> 1) == 2 ? u.z : u.w;
    w = (i & 1) ? ((w & 0x0000FFFFu) | (bits(v) << 16)) : ((w & 0xFFFF0000u) | bits(v));
  }
  static __device__ __forceinline__ void set(uint2& u, int i, float v) {
    uint32_t& w = (i >> 1) ? u.y : u.x;
    w = (i & 1) ? ((w & 0x0000FFFFu) | (bits(v) << 16)) : ((w & 0xFFFF0000u) | bits(v));
  }
};
template <> struct Pk<float> {
  static __device__ __forceinline__ float get(const uint4& u, int i) {
    return __uint_as_float(i == 0 ? u.x : i == 1 ? u.y : i == 2 ? u.z : u.w);
  }
  static __device__ __forceinline__ float get(const uint2& u, int i) { return __uint_as_float(i ? u.y : u.x); }
  static __device__ __forceinline__ void set(uint4& u, int i, float v) {
    uint32_t& w = i == 0 ? u.x : i == 1 ? u.y : i == 2 ? u.z : u.w;
    w = __float_as_uint(v);
  }
  static __device__ __forceinline__ void set(uint2& u, int i, float v) {
    uint32_t& w = i ? u.y : u.x;
    w = __float_as_uint(v);
  }
};

// ------------------------------------------------------------------------------ chain bookkeeping

struct Chain {
  int k;            // direction slab
  bool vert, rev;   // orientation; reversed step order in canonical coordinates (B2T, R2L)
  int64_t bc, chain, wplane;
  int L, P, ntiles;
};

__device__ __forceinline__ Chain make_chain(const ScanParams& p, int K, int64_t w) {
  Chain ch;
  const int64_t bc = w / p.D;
  ch.k = static_cast<int>(w % p.D);
  const uint32_t dir = p.dirbit[ch.k];
  ch.vert = (dir == GSPN_DIR_T2B) || (dir == GSPN_DIR_B2T);
  ch.rev = (dir == GSPN_DIR_B2T) || (dir == GSPN_DIR_R2L);
  ch.bc = bc;
  const int64_t b = bc / p.C, c = bc % p.C, g = c / (p.C / p.G);
  ch.chain = (ch.k * p.B + b) * p.C + c;
  ch.wplane = (ch.k * p.B + b) * p.G + g;
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
__device__ __forceinline__ void issue_tile(const StreamArgs& A, const Chain& ch, int j, int t, uint32_t st,
                                           uint32_t fb, uint64_t pol) {
  const Plan& pl = A.plan;
  const int o = ch.vert ? 0 : 1;
  const int s0 = tile_start(ch, j, pl.K);
  const int plane = static_cast<int>(plane_of<kBwd>(ch, t));
  // h_{t-1} view for the backward, one step against the scan direction (its zero fill is
  // h_{-1} = 0). Vertical: the row coordinate shifts by one. Horizontal: TMA needs a 16-byte
  // aligned inner coordinate, so a 2K-step box [s0-K, s0+K) (L2R) / [s0, s0+2K) (R2L) is
  // loaded with a 32-byte swizzle and the consumer picks element K+kk-1 / kk+1.
  const bool hview = kBwd && t == B_H;
  const uint32_t dst = st + t * pl.tile_bytes;
  if (ch.vert) {
    const int row = s0 + (hview ? (ch.rev ? 1 : -1) : 0);
    for (int q = 0; q < pl.nbw; ++q)
      tma_load3(dst + q * pl.K * pl.bw * pl.es, &A.in[o][t], q * pl.bw, row, plane, fb, pol);
  } else if (hview) {
    const int c0h = ch.rev ? s0 : s0 - pl.K;
    for (int q = 0; q < pl.nbh; ++q) tma_load3(dst + q * pl.bh * 32, &A.in[o][t], c0h, q * pl.bh, plane, fb, pol);
  } else {
    for (int q = 0; q < pl.nbh; ++q) tma_load3(dst + q * pl.bh * 16, &A.in[o][t], s0, q * pl.bh, plane, fb, pol);
  }
}

// The producer thread. Horizontal tiles are 16-byte row chunks: two consecutive tiles share every
// 32-byte DRAM sector, so with a ring of >= 3 stages they are loaded as a pair, back to back, and
// each sector is fetched from DRAM once (no reliance on L2 keeping it for a whole tile).
template <bool kBwd>
__device__ void producer_loop(const StreamArgs& A, uint8_t* ring, uint64_t* full, uint64_t* empty) {
  const Plan& pl = A.plan;
  const ScanParams& p = A.p;
  const uint64_t pol_xin = policy_of(pl.pol[0]);
  const uint64_t pol_vin = policy_of(pl.pol[1]);
  const uint64_t pol_hin = policy_of(pl.pol[2]);
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t w = blockIdx.x; w < pl.nchains; w += gridDim.x) {
    const Chain ch = make_chain(p, pl.K, w);
    for (int jj = 0; jj < ch.ntiles;) {
      const int ng = (!ch.vert && pl.pair && jj + 1 < ch.ntiles) ? 2 : 1;
      int stg[2], jt[2];
      for (int u = 0; u < ng; ++u) {
        if (pl.nosleep) mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
        else mbar_wait_sleep(smem_u32(&empty[stage]), phase ^ 1);
        mbar_arrive_tx(smem_u32(&full[stage]), ch.vert ? pl.tx_v : pl.tx_h);
        stg[u] = stage;
        jt[u] = kBwd ? (ch.ntiles - 1 - (jj + u)) : (jj + u);
        if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
      }
      for (int t = 0; t < pl.nin; ++t) {
        // x is re-read by the plane's other directions; vertical streams are read exactly once
        const uint64_t pol = t == 0 ? pol_xin : (ch.vert ? pol_vin : pol_hin);
        for (int u = 0; u < ng; ++u)
          issue_tile<kBwd>(A, ch, jt[u], t, smem_u32(ring + static_cast<size_t>(stg[u]) * pl.stage_bytes),
                           smem_u32(&full[stg[u]]), pol);
      }
      jj += ng;
    }
  }
}

// The storer thread: once the consumer warps of a horizontal tile have written its outputs in place
// (over the consumed input rows) it stores them with TMA, waits until the bulk copy has read shared
// memory, and only then hands the stage back to the producer. Vertical tiles store from registers,
// so their stage is released as soon as the consumers are done with it.
__device__ void storer_loop(const StreamArgs& A, uint8_t* ring, uint64_t* done, uint64_t* empty, int nout,
                            const int* slots, bool bwd) {
  const Plan& pl = A.plan;
  const uint64_t pol = policy_of(pl.pol[4]);
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t w = blockIdx.x; w < pl.nchains; w += gridDim.x) {
    const Chain ch = make_chain(A.p, pl.K, w);
    for (int jj = 0; jj < ch.ntiles; ++jj) {
      const int j = bwd ? (ch.ntiles - 1 - jj) : jj;
      mbar_wait(smem_u32(&done[stage]), phase);
      if (!ch.vert) {
        const int s0 = tile_start(ch, j, pl.K);
        const uint8_t* st = ring + static_cast<size_t>(stage) * pl.stage_bytes;
        for (int t = 0; t < nout; ++t) {
          const int64_t plane = t == 0 ? ch.chain : ch.wplane;
          const uint32_t src = smem_u32(st + static_cast<size_t>(slots[t]) * pl.tile_bytes);
          for (int q = 0; q < pl.nbh; ++q)
            tma_store3(&A.out[1][t], src + q * pl.bh * 16, s0, q * pl.bh, static_cast<int>(plane), pol);
        }
        bulk_commit();
        bulk_wait_read0();
      }
      mbar_arrive(smem_u32(&empty[stage]));
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
    }
  }
  bulk_wait_all();
}

// ------------------------------------------------------------------------------ per-lane geometry

// E consecutive elements of T in shared memory <-> floats (E = 2: 4/8 bytes, E = 4: 8/16 bytes).
template <typename T, int E> struct VE;
template <typename T> struct VE<T, 4> {
  static __device__ __forceinline__ void load(const uint8_t* p, float (&v)[4]) { V4<T>::load(p, v); }
  static __device__ __forceinline__ void store(uint8_t* p, const float (&v)[4]) { V4<T>::store(p, v); }
};
template <> struct VE<__nv_bfloat16, 2> {
  static __device__ __forceinline__ void load(const uint8_t* p, float (&v)[2]) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
    v[0] = __uint_as_float(u << 16);
    v[1] = __uint_as_float(u & 0xFFFF0000u);
  }
  static __device__ __forceinline__ void store(uint8_t* p, const float (&v)[2]) {
    *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(v[0], v[1]);
  }
};
template <> struct VE<float, 2> {
  static __device__ __forceinline__ void load(const uint8_t* p, float (&v)[2]) {
    const float2 u = *reinterpret_cast<const float2*>(p);
    v[0] = u.x;
    v[1] = u.y;
  }
  static __device__ __forceinline__ void store(uint8_t* p, const float (&v)[2]) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  }
};

// E consecutive outputs (E = 2 or 4) from registers straight to global memory (vertical chains:
// a warp's owned positions are contiguous, so these stores coalesce).
template <typename T, int E> struct GStore;
template <> struct GStore<__nv_bfloat16, 2> {
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float (&v)[2], uint64_t pol) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
    st_global_b32(p, *reinterpret_cast<uint32_t*>(&a), pol);
  }
};
template <> struct GStore<__nv_bfloat16, 4> {
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float (&v)[4], uint64_t pol) {
    const uint2 u = V4<__nv_bfloat16>::pack(v);
    st_global_v2(p, u.x, u.y, pol);
  }
};
template <> struct GStore<float, 2> {
  static __device__ __forceinline__ void st(float* p, const float (&v)[2], uint64_t pol) {
    st_global_v2(p, __float_as_uint(v[0]), __float_as_uint(v[1]), pol);
  }
};
template <> struct GStore<float, 4> {
  static __device__ __forceinline__ void st(float* p, const float (&v)[4], uint64_t pol) {
    st_global_v4(p, __float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3]), pol);
  }
};

template <int E>
__device__ __forceinline__ void red_add_vec(float* p, const float (&v)[E], uint64_t pol) {
  if constexpr (E == 4) red_add_v4(p, v[0], v[1], v[2], v[3], pol);
  else red_add_v2(p, v[0], v[1], pol);
}

// The E positions a lane computes, their masks, and where they live in a shared-memory tile.
// Warp w covers positions [A, A + 32 E), A = w * OWN - GH, OWN = 32 E - 2 GH; it owns the middle
// [A + GH, A + 32 E - GH) and recomputes GH ghost positions on each side.
//   vertical:   lane owns positions A + E lane + e            (e = 0..E-1)
//   horizontal: lane owns positions A + 32 e + lane           (e = slot 0..E-1)
template <int E>
struct Lanes {
  int A;
  int pos[E];
  bool valid[E], hl[E], hr[E], own[E];
  uint32_t voff;      // vertical: byte offset of the lane's E positions at kk = 0
  uint32_t vstep;     // vertical: bytes between consecutive kk
  uint32_t row[E];    // horizontal: clamped row index of each slot
};

template <typename T, int E>
__device__ __forceinline__ Lanes<E> make_lanes(const Plan& pl, const Chain& ch, int wi, int lane) {
  using C = Cfg<T>;
  constexpr int WARP = 32 * E, OWN = WARP - 2 * C::GH;
  Lanes<E> ln;
  ln.A = wi * OWN - C::GH;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int off = ch.vert ? (E * lane + e) : (32 * e + lane);
    const int r = ln.A + off;
    ln.pos[e] = r;
    ln.valid[e] = (r >= 0) && (r < ch.P);
    ln.hl[e] = r >= 1;
    ln.hr[e] = r <= ch.P - 2;
    // owned, and inside the tile (positions >= ppad are padding >= P: nothing to store)
    ln.own[e] = (off >= C::GH) && (off < WARP - C::GH) && (r < pl.ppad);
    const int rc = r < 0 ? 0 : (r >= pl.ppad ? pl.ppad - 1 : r);
    ln.row[e] = static_cast<uint32_t>(rc);
  }
  int r0 = ln.A + E * lane;
  r0 = r0 < 0 ? 0 : (r0 > pl.ppad - E ? pl.ppad - E : r0);
  const int bwl = 31 - __clz(pl.bw);
  ln.voff = static_cast<uint32_t>((((r0 >> bwl) * C::K) * pl.bw + (r0 & (pl.bw - 1))) * C::es);
  ln.vstep = static_cast<uint32_t>(pl.bw * C::es);
  return ln;
}

// Ghost exchange at a tile boundary. Each warp publishes its first GH and last GH owned values
// (edges) and reloads its ghost positions from the neighbouring warps' edges; warps outside
// [0, nwc) contribute 0. Parity-double-buffered; the caller separates publish and reload by a barrier.
template <typename T, int E>
__device__ __forceinline__ void edge_publish(float* edge, int par, int wi, int lane, bool vert, const float (&v)[E]) {
  using C = Cfg<T>;
  constexpr int WARP = 32 * E;
  float* L = edge + ((par * kEdgeW + wi) * 2 + 0) * 8;
  float* R = edge + ((par * kEdgeW + wi) * 2 + 1) * 8;
  if (vert) {
    const int o = E * lane;
    if (o >= C::GH && o < 2 * C::GH) {
#pragma unroll
      for (int e = 0; e < E; ++e) L[o - C::GH + e] = v[e];
    }
    if (o >= WARP - 2 * C::GH && o < WARP - C::GH) {
#pragma unroll
      for (int e = 0; e < E; ++e) R[o - (WARP - 2 * C::GH) + e] = v[e];
    }
  } else {
    if (lane >= C::GH && lane < 2 * C::GH) L[lane - C::GH] = v[0];
    if (lane >= 32 - 2 * C::GH && lane < 32 - C::GH) R[lane - (32 - 2 * C::GH)] = v[E - 1];
  }
}

template <typename T, int E>
__device__ __forceinline__ void edge_reload(const float* edge, int par, int wi, int nwc, int lane, bool vert,
                                            float (&v)[E]) {
  using C = Cfg<T>;
  constexpr int WARP = 32 * E;
  const float* Rl = edge + ((par * kEdgeW + (wi - 1)) * 2 + 1) * 8;  // left neighbour's right edge
  const float* Lr = edge + ((par * kEdgeW + (wi + 1)) * 2 + 0) * 8;  // right neighbour's left edge
  if (vert) {
    const int o = E * lane;
    if (o < C::GH) {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = wi > 0 ? Rl[o + e] : 0.f;
    }
    if (o >= WARP - C::GH) {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = wi < nwc - 1 ? Lr[o - (WARP - C::GH) + e] : 0.f;
    }
  } else {
    if (lane < C::GH) v[0] = wi > 0 ? Rl[lane] : 0.f;
    if (lane >= 32 - C::GH) v[E - 1] = wi < nwc - 1 ? Lr[lane - (32 - C::GH)] : 0.f;
  }
}

// Neighbours inside a warp. Vertical (blocked): position e's lower neighbour is e-1 of the same lane
// (lane-1's last for e = 0); horizontal (interleaved, position A + 32 q + lane): one rotating
// shuffle per slot; lane 0 of slot q takes lane 31 of slot q-1, lane 31 takes lane 0 of slot q+1.
// The warp's two outermost positions get 0 (they are ghosts).
template <int E>
__device__ __forceinline__ void vert_neighbours(const float (&v)[E], int lane, float (&lo)[E], float (&hi)[E]) {
  const float left = from_lower_lane(v[E - 1], lane);
  const float right = from_upper_lane(v[0], lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    lo[e] = e == 0 ? left : v[e > 0 ? e - 1 : 0];
    hi[e] = e == E - 1 ? right : v[e < E - 1 ? e + 1 : 0];
  }
}

template <int E>
__device__ __forceinline__ void slot_neighbours(const float (&v)[E], int lane, float (&lo)[E], float (&hi)[E]) {
  float up[E], dn[E];
#pragma unroll
  for (int q = 0; q < E; ++q) {
    up[q] = __shfl_sync(0xffffffffu, v[q], (lane + 31) & 31);
    dn[q] = __shfl_sync(0xffffffffu, v[q], (lane + 1) & 31);
  }
#pragma unroll
  for (int q = 0; q < E; ++q) {
    lo[q] = lane == 0 ? (q == 0 ? 0.f : up[q > 0 ? q - 1 : 0]) : up[q];
    hi[q] = lane == 31 ? (q == E - 1 ? 0.f : dn[q < E - 1 ? q + 1 : 0]) : dn[q];
  }
}

// Element-order reversal of packed row chunks (runtime flag), so horizontal chains of both
// directions see their steps in scan order: after it, element s of a row chunk is in-tile step s.
__device__ __forceinline__ uint32_t swap16(uint32_t v) { return __byte_perm(v, 0, 0x1032); }
template <typename T> struct Rev;
template <> struct Rev<__nv_bfloat16> {
  static __device__ __forceinline__ uint4 r(const uint4& u, bool rev) {
    return rev ? make_uint4(swap16(u.w), swap16(u.z), swap16(u.y), swap16(u.x)) : u;
  }
  static __device__ __forceinline__ uint2 r(const uint2& u, bool rev) {
    return rev ? make_uint2(swap16(u.y), swap16(u.x)) : u;
  }
};
template <> struct Rev<float> {
  static __device__ __forceinline__ uint4 r(const uint4& u, bool rev) { return rev ? make_uint4(u.w, u.z, u.y, u.x) : u; }
  static __device__ __forceinline__ uint2 r(const uint2& u, bool rev) { return rev ? make_uint2(u.y, u.x) : u; }
};

// ------------------------------------------------------------------------------ forward consumer

// One step of Eq. 1 for the lane's E positions given the previous state's neighbours.
template <int E>
__device__ __forceinline__ void fwd_update(const Lanes<E>& ln, const float (&x)[E], const float (&lam)[E],
                                           const float (&wl)[E], const float (&wm)[E], const float (&wr)[E],
                                           const float (&hm1)[E], const float (&hp1)[E], float (&h)[E],
                                           bool prenorm) {
  float hn[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const float l = ln.hl[e] ? wl[e] : 0.f;
    const float r = ln.hr[e] ? wr[e] : 0.f;
    const float acc = fmaf(l, hm1[e], fmaf(wm[e], h[e], r * hp1[e]));
    const float inv = prenorm ? 1.f : fast_rcp(wm[e] + l + r);
    hn[e] = ln.valid[e] ? fmaf(acc, inv, lam[e] * x[e]) : 0.f;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) h[e] = hn[e];
}

// Vertical tile: the step loop stays rolled (code size); the in-tile row is a runtime offset. The
// new state goes from registers straight to global memory (coalesced: a warp's owned positions
// are contiguous).
template <typename T, int E>
__device__ __forceinline__ void fwd_tile_vert(const Plan& pl, const Lanes<E>& ln, const Chain& ch, int j,
                                              const uint8_t* st, T* hplane, int64_t W, int lane, float (&h)[E],
                                              bool prenorm, uint64_t pol) {
  constexpr int K = Cfg<T>::K;
  const bool rev = ch.rev;
  const int dk = rev ? -static_cast<int>(ln.vstep) : static_cast<int>(ln.vstep);
  uint32_t off = ln.voff + (rev ? (K - 1) * ln.vstep : 0u);
  const bool lane_out = ln.own[0] && ln.valid[0];  // P % E == 0: a lane's positions share validity
#pragma unroll 1
  for (int s = 0; s < K; ++s, off += dk) {
    float x[E], lam[E], wl[E], wm[E], wr[E], hm1[E], hp1[E];
    VE<T, E>::load(st + F_X * pl.tile_bytes + off, x);
    VE<T, E>::load(st + F_LAM * pl.tile_bytes + off, lam);
    VE<T, E>::load(st + F_WL * pl.tile_bytes + off, wl);
    VE<T, E>::load(st + F_WM * pl.tile_bytes + off, wm);
    VE<T, E>::load(st + F_WR * pl.tile_bytes + off, wr);
    vert_neighbours<E>(h, lane, hm1, hp1);
    fwd_update<E>(ln, x, lam, wl, wm, wr, hm1, hp1, h, prenorm);
    const int t = j * K + s;
    if (lane_out && t < ch.L) {
      const int row = rev ? (ch.L - 1 - t) : t;
      GStore<T, E>::st(hplane + static_cast<int64_t>(row) * W + ln.pos[0], h, pol);
    }
  }
}

// Horizontal tile: one 16-byte row chunk (K steps) per tensor per slot, put in scan order. Once every
// consumer warp holds its rows in registers (named barrier), the new state is written in place over
// the consumed x rows, from where the storer warp sends the tile out with TMA.
template <typename T, int E>
__device__ __forceinline__ void fwd_tile_horiz(const Plan& pl, const Lanes<E>& ln, uint8_t* st, int lane, bool rev,
                                               float (&h)[E], bool prenorm, int nthreads) {
  constexpr int K = Cfg<T>::K;
  uint4 X[E], LAM[E], WL[E], WM[E], WR[E], OUT[E];
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const uint32_t off = ln.row[q] * 16;
    X[q] = Rev<T>::r(*reinterpret_cast<const uint4*>(st + F_X * pl.tile_bytes + off), rev);
    LAM[q] = Rev<T>::r(*reinterpret_cast<const uint4*>(st + F_LAM * pl.tile_bytes + off), rev);
    WL[q] = Rev<T>::r(*reinterpret_cast<const uint4*>(st + F_WL * pl.tile_bytes + off), rev);
    WM[q] = Rev<T>::r(*reinterpret_cast<const uint4*>(st + F_WM * pl.tile_bytes + off), rev);
    WR[q] = Rev<T>::r(*reinterpret_cast<const uint4*>(st + F_WR * pl.tile_bytes + off), rev);
    OUT[q] = make_uint4(0, 0, 0, 0);
  }
  named_bar(kBarRows, nthreads);  // all rows (incl. other warps' ghost rows) are in registers now
#pragma unroll
  for (int s = 0; s < K; ++s) {
    float hm1[E], hp1[E], x[E], lam[E], wl[E], wm[E], wr[E];
    slot_neighbours<E>(h, lane, hm1, hp1);
#pragma unroll
    for (int q = 0; q < E; ++q) {
      x[q] = Pk<T>::get(X[q], s);
      lam[q] = Pk<T>::get(LAM[q], s);
      wl[q] = Pk<T>::get(WL[q], s);
      wm[q] = Pk<T>::get(WM[q], s);
      wr[q] = Pk<T>::get(WR[q], s);
    }
    fwd_update<E>(ln, x, lam, wl, wm, wr, hm1, hp1, h, prenorm);
#pragma unroll
    for (int q = 0; q < E; ++q) Pk<T>::set(OUT[q], s, h[q]);
  }
#pragma unroll
  for (int q = 0; q < E; ++q)
    if (ln.own[q]) *reinterpret_cast<uint4*>(st + F_X * pl.tile_bytes + ln.row[q] * 16) = Rev<T>::r(OUT[q], rev);
}

// Shared-memory carve-up common to both kernels: ring | full | empty | done | edges | flag.
struct Smem {
  uint8_t* ring;
  uint64_t *full, *empty, *done;
  float* edge;
  int* flag;
};

__device__ __forceinline__ Smem carve(uint8_t* smem_raw, const Plan& pl) {
  Smem m;
  m.ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared space
  m.full = reinterpret_cast<uint64_t*>(m.ring + static_cast<size_t>(pl.nstages) * pl.stage_bytes);
  m.empty = m.full + pl.nstages;
  m.done = m.empty + pl.nstages;
  m.edge = reinterpret_cast<float*>(m.done + pl.nstages);  // [3 state arrays][2 par][kEdgeW][2][8]
  m.flag = reinterpret_cast<int*>(m.edge + 3 * 2 * kEdgeW * 2 * 8);
  return m;
}

__device__ __forceinline__ void init_barriers(const Smem& m, const Plan& pl) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < pl.nstages; ++s) {
      mbar_init(smem_u32(&m.full[s]), 1);       // producer arrive + TMA bytes
      mbar_init(smem_u32(&m.empty[s]), 1);      // storer
      mbar_init(smem_u32(&m.done[s]), pl.nwc);  // one arrive per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

template <typename T, int E, int kMaxNWC>
__global__ void __launch_bounds__((kMaxNWC + 2) * 32, kMaxNWC <= 6 ? 2 : 1)
    fwd_stream_kernel(const __grid_constant__ StreamArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Plan& pl = A.plan;
  const Smem m = carve(smem_raw, pl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  init_barriers(m, pl);
  if (warp == pl.nwc) {  // producer warp
    if (lane == 0) {
      for (int o = 0; o < 2; ++o)
        for (int t = 0; t < F_NIN; ++t) asm volatile("prefetch.tensormap [%0];" ::"l"(&A.in[o][t]) : "memory");
      producer_loop<false>(A, m.ring, m.full, m.empty);
    }
    return;
  }
  if (warp == pl.nwc + 1) {  // storer warp
    if (lane == 0) {
      const int slots[1] = {F_X};
      storer_loop(A, m.ring, m.done, m.empty, 1, slots, false);
    }
    return;
  }
  const bool prenorm = A.p.flags & GSPN_FLAG_PRENORMALIZED;
  const uint64_t pol_vout = policy_of(pl.pol[3]);
  const int nthreads = pl.nwc * 32;
  const int64_t HW = A.p.H * A.p.W;
  int stage = 0, par = 0;
  uint32_t phase = 0;
  for (int64_t w = blockIdx.x; w < pl.nchains; w += gridDim.x) {
    const Chain ch = make_chain(A.p, pl.K, w);
    const Lanes<E> ln = make_lanes<T, E>(pl, ch, warp, lane);
    T* hplane = static_cast<T*>(A.p.hout) + ch.chain * HW;
    float h[E];
#pragma unroll
    for (int e = 0; e < E; ++e) h[e] = 0.f;
    for (int j = 0; j < ch.ntiles; ++j) {
      mbar_wait(smem_u32(&m.full[stage]), phase);
      uint8_t* st = m.ring + static_cast<size_t>(stage) * pl.stage_bytes;
      if (pl.null_compute) {
      } else if (ch.vert) {
        fwd_tile_vert<T, E>(pl, ln, ch, j, st, hplane, A.p.W, lane, h, prenorm, pol_vout);
      } else {
        fwd_tile_horiz<T, E>(pl, ln, st, lane, ch.rev, h, prenorm, nthreads);
      }
      fence_proxy_async();  // in-place outputs -> visible to the storer's TMA (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&m.done[stage]));
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
      edge_publish<T, E>(m.edge, par, warp, lane, ch.vert, h);
      named_bar(kBarTile, nthreads);
      edge_reload<T, E>(m.edge, par, warp, pl.nwc, lane, ch.vert, h);
      par ^= 1;
    }
  }
}

// ------------------------------------------------------------------------------ backward consumer

// State carried between steps (reverse order): ea = a_{t+1} g_{t+1}, eb = b_{t+1} g_{t+1},
// ec = c_{t+1} g_{t+1} at the lane's E positions.
template <int E>
struct BwdState {
  float ea[E], eb[E], ec[E];
};

// One adjoint step for the lane's E positions. nr/nl: (a g) of the upper neighbour / (c g) of the
// lower neighbour; hm1/h0/hp1: h_{t-1} at r-1, r, r+1. Outputs dlam, dw (or the tap gradients D for
// the grouped path), dxv = g lam; the state is replaced by step t's products. Per-channel weights
// get the normalisation Jacobian in the cancellation-free form (gspn_common.cuh: jacobian), written
// with u = h[r-1] - h[r], v = h[r+1] - h[r]:
//   dw_l = g ((m + r) u - r v) / S^2,  dw_m = -g (l u + r v) / S^2,  dw_r = g ((l + m) v - l u) / S^2.
template <int E, bool kGrouped>
__device__ __forceinline__ void bwd_update(const Lanes<E>& ln, bool live, const float (&x)[E], const float (&lam)[E],
                                           const float (&dh)[E], const float (&wl)[E], const float (&wm)[E],
                                           const float (&wr)[E], const float (&hm1)[E], const float (&h0)[E],
                                           const float (&hp1)[E], const float (&nr)[E], const float (&nl)[E],
                                           BwdState<E>& S, float (&dlam)[E], float (&o1)[E], float (&o2)[E],
                                           float (&o3)[E], float (&dxv)[E], bool prenorm) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const bool ok = live && ln.valid[e];
    const float g = ok ? (dh[e] + S.eb[e] + nr[e] + nl[e]) : 0.f;
    const float l = ln.hl[e] ? wl[e] : 0.f;
    const float r = ln.hr[e] ? wr[e] : 0.f;
    const float inv = prenorm ? 1.f : fast_rcp(wm[e] + l + r);
    const float ig = inv * g;
    dlam[e] = g * x[e];
    dxv[e] = g * lam[e];
    if (kGrouped || prenorm) {
      o1[e] = ln.hl[e] ? g * hm1[e] : 0.f;
      o2[e] = g * h0[e];
      o3[e] = ln.hr[e] ? g * hp1[e] : 0.f;
    } else {
      const float q = ig * inv;
      const float u = hm1[e] - h0[e], v = hp1[e] - h0[e];
      const float rv = r * v, lu = l * u;
      o1[e] = ln.hl[e] ? q * fmaf(wm[e] + r, u, -rv) : 0.f;
      o2[e] = -q * (lu + rv);
      o3[e] = ln.hr[e] ? q * fmaf(l + wm[e], v, -lu) : 0.f;
    }
    S.ea[e] = ok ? l * ig : 0.f;
    S.eb[e] = ok ? wm[e] * ig : 0.f;
    S.ec[e] = ok ? r * ig : 0.f;
  }
}

template <typename T, int E, bool kGrouped>
__device__ __forceinline__ void bwd_tile_vert(const StreamArgs& A, const Lanes<E>& ln, const Chain& ch, int j,
                                              const uint8_t* st, int lane, BwdState<E>& S, bool prenorm,
                                              uint64_t pol_acc, uint64_t pol_out) {
  constexpr int K = Cfg<T>::K;
  const Plan& pl = A.plan;
  const ScanParams& p = A.p;
  const int64_t HW = p.H * p.W;
  float* dxacc = p.dx_acc + ch.bc * HW;
  const int64_t wofs = ch.wplane * HW;
  const bool lane_out = ln.own[0] && ln.valid[0];  // P % E == 0: a lane's positions share validity
  // steps s = K-1 .. 0 (reverse); in-tile row kk = rev ? K-1-s : s
  const int dk = ch.rev ? static_cast<int>(ln.vstep) : -static_cast<int>(ln.vstep);
  uint32_t off = ln.voff + (ch.rev ? 0u : (K - 1) * ln.vstep);
#pragma unroll 1
  for (int s = K - 1; s >= 0; --s, off += dk) {
    const int t = j * K + s;
    const bool live = t < ch.L;
    float x[E], lam[E], dh[E], wl[E], wm[E], wr[E], hp[E], hm1[E], hp1[E], nr[E], nl[E], lo_a[E], hi_c[E];
    VE<T, E>::load(st + B_X * pl.tile_bytes + off, x);
    VE<T, E>::load(st + B_LAM * pl.tile_bytes + off, lam);
    VE<T, E>::load(st + B_DH * pl.tile_bytes + off, dh);
    VE<T, E>::load(st + B_WL * pl.tile_bytes + off, wl);
    VE<T, E>::load(st + B_WM * pl.tile_bytes + off, wm);
    VE<T, E>::load(st + B_WR * pl.tile_bytes + off, wr);
    VE<T, E>::load(st + B_H * pl.tile_bytes + off, hp);
    vert_neighbours<E>(hp, lane, hm1, hp1);
    vert_neighbours<E>(S.ea, lane, lo_a, nr);   // nr[e] = (a g) of position e + 1
    vert_neighbours<E>(S.ec, lane, nl, hi_c);   // nl[e] = (c g) of position e - 1
    float dlam[E], o1[E], o2[E], o3[E], dxv[E];
    bwd_update<E, kGrouped>(ln, live, x, lam, dh, wl, wm, wr, hm1, hp, hp1, nr, nl, S, dlam, o1, o2, o3, dxv, prenorm);
    if (lane_out && live) {
      const int row = ch.rev ? (ch.L - 1 - t) : t;
      const int64_t o = static_cast<int64_t>(row) * p.W + ln.pos[0];
      GStore<T, E>::st(static_cast<T*>(p.dlam) + ch.chain * HW + o, dlam, pol_out);
      if (!kGrouped) {
        GStore<T, E>::st(static_cast<T*>(p.dwl) + wofs + o, o1, pol_out);
        GStore<T, E>::st(static_cast<T*>(p.dwm) + wofs + o, o2, pol_out);
        GStore<T, E>::st(static_cast<T*>(p.dwr) + wofs + o, o3, pol_out);
      }
      red_add_vec<E>(dxacc + o, dxv, pol_acc);
      if (kGrouped && t >= 1) {
        red_add_vec<E>(p.dwa_l + wofs + o, o1, pol_acc);
        red_add_vec<E>(p.dwa_m + wofs + o, o2, pol_acc);
        red_add_vec<E>(p.dwa_r + wofs + o, o3, pol_acc);
      }
    }
  }
}

// Horizontal backward tile. Rows of x, lam, dh and the taps come in as 16-byte chunks (K steps,
// put in scan order); they are processed as NSUB sub-tiles of KS steps (the upper half first: the
// backward walks the steps downwards) with the working half selected at run time, which keeps one
// copy of the unrolled step code. h_{t-1} is read per step from the 2K-step swizzled h row.
template <typename T, int E, bool kGrouped>
__device__ __forceinline__ void bwd_tile_horiz(const StreamArgs& A, const Lanes<E>& ln, const Chain& ch, int j,
                                               uint8_t* st, int lane, BwdState<E>& S, bool prenorm,
                                               uint64_t pol_acc, int nthreads) {
  using C = Cfg<T>;
  constexpr int K = C::K, KS = C::KS, NSUB = K / KS;
  static_assert(NSUB == 2, "sub-tiles are the two 8-byte halves of a 16-byte row chunk");
  const Plan& pl = A.plan;
  const ScanParams& p = A.p;
  const bool rev = ch.rev;
  const int64_t HW = p.H * p.W;
  float* dxacc = p.dx_acc + ch.bc * HW;
  const int64_t wofs = ch.wplane * HW;
  const int c0 = tile_start(ch, j, K);  // canonical column of kk = 0 (W % K == 0 on this path)
  const uint8_t* hbase = st + B_H * pl.tile_bytes;
  uint4 X[E], LAM[E], DH[E], WL[E], WM[E], WR[E];
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const uint32_t off = ln.row[q] * 16;
    X[q] = Rev<T>::r(*reinterpret_cast<const uint4*>(st + B_X * pl.tile_bytes + off), rev);
    LAM[q] = Rev<T>::r(*reinterpret_cast<const uint4*>(st + B_LAM * pl.tile_bytes + off), rev);
    DH[q] = Rev<T>::r(*reinterpret_cast<const uint4*>(st + B_DH * pl.tile_bytes + off), rev);
    WL[q] = Rev<T>::r(*reinterpret_cast<const uint4*>(st + B_WL * pl.tile_bytes + off), rev);
    WM[q] = Rev<T>::r(*reinterpret_cast<const uint4*>(st + B_WM * pl.tile_bytes + off), rev);
    WR[q] = Rev<T>::r(*reinterpret_cast<const uint4*>(st + B_WR * pl.tile_bytes + off), rev);
  }
  // every consumer warp holds its rows in registers: outputs may now overwrite x and the taps in place
  named_bar(kBarRows, nthreads);
  uint8_t* ob = st;  // dlam -> x slot, dw_l/m/r -> w_l/m/r slots (O_* == B_* slot indices below)
#pragma unroll 1
  for (int sub = NSUB - 1; sub >= 0; --sub) {
    uint2 x2[E], lam2[E], dh2[E], wl2[E], wm2[E], wr2[E];
#pragma unroll
    for (int q = 0; q < E; ++q) {
      x2[q] = sub ? make_uint2(X[q].z, X[q].w) : make_uint2(X[q].x, X[q].y);
      lam2[q] = sub ? make_uint2(LAM[q].z, LAM[q].w) : make_uint2(LAM[q].x, LAM[q].y);
      dh2[q] = sub ? make_uint2(DH[q].z, DH[q].w) : make_uint2(DH[q].x, DH[q].y);
      wl2[q] = sub ? make_uint2(WL[q].z, WL[q].w) : make_uint2(WL[q].x, WL[q].y);
      wm2[q] = sub ? make_uint2(WM[q].z, WM[q].w) : make_uint2(WM[q].x, WM[q].y);
      wr2[q] = sub ? make_uint2(WR[q].z, WR[q].w) : make_uint2(WR[q].x, WR[q].y);
    }
    uint2 OL[E], O1[E], O2[E], O3[E];
    float DXa[E][KS], DA[E][KS], DB[E][KS], DC[E][KS];
#pragma unroll
    for (int q = 0; q < E; ++q) OL[q] = O1[q] = O2[q] = O3[q] = make_uint2(0, 0);
#pragma unroll
    for (int ss = KS - 1; ss >= 0; --ss) {
      const int s = sub * KS + ss;  // in-tile step (scan order)
      const int t = j * K + s;
      // h_{t-1}: element K + s - 1 (L2R) / K - s (R2L) of the canonical 2K-step h row, whose 16-byte
      // chunks are swizzled by row bit 2 (TMA SWIZZLE_32B)
      const int he = rev ? (K - s) : (K + s - 1);
      float x[E], lam[E], dh[E], wl[E], wm[E], wr[E], h0[E];
#pragma unroll
      for (int q = 0; q < E; ++q) {
        x[q] = Pk<T>::get(x2[q], ss);
        lam[q] = Pk<T>::get(lam2[q], ss);
        dh[q] = Pk<T>::get(dh2[q], ss);
        wl[q] = Pk<T>::get(wl2[q], ss);
        wm[q] = Pk<T>::get(wm2[q], ss);
        wr[q] = Pk<T>::get(wr2[q], ss);
        const uint32_t r = ln.row[q];
        const uint32_t c16 = static_cast<uint32_t>(he / K) ^ ((r >> 2) & 1);
        h0[q] = to_f(*reinterpret_cast<const T*>(hbase + r * 32 + (c16 << 4) + (he % K) * C::es));
      }
      float hm1[E], hp1[E], nr[E], nl[E], ea_lo[E], ec_hi[E];
      slot_neighbours<E>(h0, lane, hm1, hp1);
      slot_neighbours<E>(S.ea, lane, ea_lo, nr);
      slot_neighbours<E>(S.ec, lane, nl, ec_hi);
      float dlam[E], o1[E], o2[E], o3[E], dxv[E];
      bwd_update<E, kGrouped>(ln, true, x, lam, dh, wl, wm, wr, hm1, h0, hp1, nr, nl, S, dlam, o1, o2, o3, dxv,
                              prenorm);
#pragma unroll
      for (int q = 0; q < E; ++q) {
        Pk<T>::set(OL[q], ss, dlam[q]);
        if (!kGrouped) {
          Pk<T>::set(O1[q], ss, o1[q]);
          Pk<T>::set(O2[q], ss, o2[q]);
          Pk<T>::set(O3[q], ss, o3[q]);
        } else {
          DA[q][ss] = t >= 1 ? o1[q] : 0.f;
          DB[q][ss] = t >= 1 ? o2[q] : 0.f;
          DC[q][ss] = t >= 1 ? o3[q] : 0.f;
        }
        DXa[q][ss] = dxv[q];
      }
    }
    // write back in canonical order: chunk c8 of the row, elements reversed for R2L
    const int c8 = rev ? (NSUB - 1 - sub) : sub;
#pragma unroll
    for (int q = 0; q < E; ++q) {
      if (!ln.own[q]) continue;
      const uint32_t off = ln.row[q] * 16 + c8 * 8;
      *reinterpret_cast<uint2*>(ob + B_X * pl.tile_bytes + off) = Rev<T>::r(OL[q], rev);
      if (!kGrouped) {
        *reinterpret_cast<uint2*>(ob + B_WL * pl.tile_bytes + off) = Rev<T>::r(O1[q], rev);
        *reinterpret_cast<uint2*>(ob + B_WM * pl.tile_bytes + off) = Rev<T>::r(O2[q], rev);
        *reinterpret_cast<uint2*>(ob + B_WR * pl.tile_bytes + off) = Rev<T>::r(O3[q], rev);
      }
      if (ln.valid[q]) {
        const int64_t o = static_cast<int64_t>(ln.pos[q]) * p.W + c0 + c8 * KS;
        float d[KS];
#pragma unroll
        for (int i = 0; i < KS; ++i) d[i] = rev ? DXa[q][KS - 1 - i] : DXa[q][i];
        red_add_vec<KS>(dxacc + o, d, pol_acc);
        if (kGrouped) {
          float* dst[3] = {p.dwa_l + wofs + o, p.dwa_m + wofs + o, p.dwa_r + wofs + o};
#pragma unroll
          for (int m = 0; m < 3; ++m) {
#pragma unroll
            for (int i = 0; i < KS; ++i) {
              const int si = rev ? KS - 1 - i : i;
              d[i] = m == 0 ? DA[q][si] : (m == 1 ? DB[q][si] : DC[q][si]);
            }
            red_add_vec<KS>(dst[m], d, pol_acc);
          }
        }
      }
    }
  }
}

// The last of a plane's D chains converts the fp32 dx accumulator and drops it from L2 (discard: no
// write-back of dead lines); the last of a group's C/G channels applies the normalisation Jacobian
// to the group-summed tap gradients.
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
    const int64_t n4 = HW / 4;
    constexpr int U = 8;  // independent L2 loads in flight per thread
    for (int64_t i0 = threadIdx.x; i0 < n4; i0 += static_cast<int64_t>(U) * nthreads) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + static_cast<int64_t>(u) * nthreads;
        v[u] = i < n4 ? __ldcg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + static_cast<int64_t>(u) * nthreads;
        if (i < n4) store4_global<T>(dst + 4 * i, v[u]);
      }
    }
    named_bar(kBarTile, nthreads);
    const char* base = reinterpret_cast<const char*>(p.dx_acc + ch.bc * HW);
    for (int64_t l = threadIdx.x; l < (HW * 4) / 128; l += nthreads) discard_l2_line(base + l * 128);
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

template <typename T, int E, bool kGrouped, int kMaxNWC>
__global__ void __launch_bounds__((kMaxNWC + 2) * 32, 1) bwd_stream_kernel(const __grid_constant__ StreamArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Plan& pl = A.plan;
  const Smem m = carve(smem_raw, pl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  init_barriers(m, pl);
  if (warp == pl.nwc) {
    if (lane == 0) {
      for (int o = 0; o < 2; ++o)
        for (int t = 0; t < B_NIN; ++t) asm volatile("prefetch.tensormap [%0];" ::"l"(&A.in[o][t]) : "memory");
      producer_loop<true>(A, m.ring, m.full, m.empty);
    }
    return;
  }
  if (warp == pl.nwc + 1) {  // storer warp (horizontal tiles' in-place outputs)
    if (lane == 0) {
      const int slots[4] = {B_X, B_WL, B_WM, B_WR};
      storer_loop(A, m.ring, m.done, m.empty, kGrouped ? 1 : 4, slots, true);
    }
    return;
  }
  const bool prenorm = A.p.flags & GSPN_FLAG_PRENORMALIZED;
  const uint64_t pol_vout = policy_of(pl.pol[3]);
  const uint64_t pol_acc = policy_of(pl.pol[5]);
  const int nthreads = pl.nwc * 32;
  constexpr int kEdgeArr = 2 * kEdgeW * 2 * 8;
  int stage = 0, par = 0;
  uint32_t phase = 0;
  for (int64_t w = blockIdx.x; w < pl.nchains; w += gridDim.x) {
    const Chain ch = make_chain(A.p, pl.K, w);
    const Lanes<E> ln = make_lanes<T, E>(pl, ch, warp, lane);
    BwdState<E> S;
#pragma unroll
    for (int e = 0; e < E; ++e) S.ea[e] = S.eb[e] = S.ec[e] = 0.f;
    for (int jj = 0; jj < ch.ntiles; ++jj) {
      const int j = ch.ntiles - 1 - jj;
      mbar_wait(smem_u32(&m.full[stage]), phase);
      uint8_t* st = m.ring + static_cast<size_t>(stage) * pl.stage_bytes;
      if (pl.null_compute) {
      } else if (ch.vert) {
        bwd_tile_vert<T, E, kGrouped>(A, ln, ch, j, st, lane, S, prenorm, pol_acc, pol_vout);
      } else {
        bwd_tile_horiz<T, E, kGrouped>(A, ln, ch, j, st, lane, S, prenorm, pol_acc, nthreads);
      }
      fence_proxy_async();  // in-place outputs -> visible to the storer's TMA (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&m.done[stage]));
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
      edge_publish<T, E>(m.edge + 0 * kEdgeArr, par, warp, lane, ch.vert, S.ea);
      edge_publish<T, E>(m.edge + 1 * kEdgeArr, par, warp, lane, ch.vert, S.eb);
      edge_publish<T, E>(m.edge + 2 * kEdgeArr, par, warp, lane, ch.vert, S.ec);
      named_bar(kBarTile, nthreads);
      edge_reload<T, E>(m.edge + 0 * kEdgeArr, par, warp, pl.nwc, lane, ch.vert, S.ea);
      edge_reload<T, E>(m.edge + 1 * kEdgeArr, par, warp, pl.nwc, lane, ch.vert, S.eb);
      edge_reload<T, E>(m.edge + 2 * kEdgeArr, par, warp, pl.nwc, lane, ch.vert, S.ec);
      par ^= 1;
    }
    bwd_chain_epilogue<T, kGrouped>(A, ch, m.flag, nthreads);
  }
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
            int box1, CUtensorMapL2promotion promote, bool swizzle32 = false) {
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
                  promote,
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

// L2 promotion of the horizontal (16-byte row chunk) TMA loads; GSPN_L2PROMO=0|64|128|256 overrides
// (experiments only). Default: none — the next tile's chunk shares the 32-byte sector anyway.
CUtensorMapL2promotion horiz_promotion() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GSPN_L2PROMO");
    v = e ? atoi(e) : 0;
  }
  switch (v) {
    case 64: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 128: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    case 256: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
  }
}

constexpr int kSmemTail = 6656;  // mbarriers (3 per stage), ghost-edge buffers (6 KB), flag

// Shape eligibility + plan. nin/nout: tensors per tile.
bool make_plan(const ScanParams& p, gspn_dtype_t dt, int nin, int nout, int min_stages, bool two_ctas, int E,
               Plan* pl) {
  const int s = dt == GSPN_BF16 ? 2 : 4;
  if ((p.W * s) % 16 != 0) return false;  // TMA global stride alignment; also K | W for horizontal tiles
  bool any_v = false, any_h = false;
  for (int k = 0; k < p.D; ++k) {
    if (p.dirbit[k] == GSPN_DIR_T2B || p.dirbit[k] == GSPN_DIR_B2T) any_v = true; else any_h = true;
  }
  const int64_t maxP = std::max<int64_t>(any_v ? p.W : 0, any_h ? p.H : 0);
  memset(pl, 0, sizeof *pl);
  pl->K = 16 / s;
  pl->es = s;
  pl->own = 32 * E - 2 * pl->K;
  pl->nwc = static_cast<int>((maxP + pl->own - 1) / pl->own);
  if (pl->nwc > kEdgeW) return false;
  // positions addressable in a tile: every owned position, a whole number of vertical boxes
  int ppad = static_cast<int>((maxP + 63) / 64 * 64);
  int bw = 0;
  for (int b = 256; b >= 16 / s; b >>= 1)
    if (ppad % b == 0 && (p.W + b - 1) / b * b <= ppad) { bw = b; break; }
  if (bw == 0) {  // round ppad up to the widest box that tiles W
    bw = 64;
    ppad = (ppad + 63) / 64 * 64;
  }
  pl->ppad = ppad;
  pl->bw = bw;
  pl->bh = 0;
  for (int b = 256; b >= 1; b >>= 1)
    if ((p.H + b - 1) / b * b <= ppad) { pl->bh = b; break; }
  if (pl->bh == 0) return false;
  pl->nbw = static_cast<int>((p.W + pl->bw - 1) / pl->bw);
  pl->nbh = static_cast<int>((p.H + pl->bh - 1) / pl->bh);
  pl->nin = nin;
  pl->nout = nout;
  pl->tile_bytes = static_cast<uint32_t>(pl->K * pl->ppad * s);
  pl->h_wide = (nin == B_NIN) ? 1 : 0;
  pl->stage_bytes = (nin + pl->h_wide) * pl->tile_bytes;
  pl->tx_v = static_cast<uint32_t>(nin * pl->nbw * pl->bw * pl->K * s);
  pl->tx_h = static_cast<uint32_t>((nin + pl->h_wide) * pl->nbh * pl->bh * pl->K * s);
  const int budget = smem_optin() - 1024 /*alignment*/ - kSmemTail;
  const int avail = budget;
  int ns = avail / static_cast<int>(pl->stage_bytes);
  // Two CTAs per SM when both fit with >= 2 stages each: the second chain hides the first's
  // per-tile latencies. Otherwise one CTA with a deeper ring.
  const int half = (smem_optin() / 2 - 1024 - kSmemTail) /
                   static_cast<int>(pl->stage_bytes);
  if (const char* e = getenv("GSPN_FWD_CTAS")) {  // experiments: force the fwd to 1 or 2 CTAs per SM
    if (two_ctas && atoi(e) == 1) two_ctas = false;
  }
  if (two_ctas && half >= 2 && pl->nwc <= 6) ns = std::min(half, 4);
  if (ns > 8) ns = 8;
  if (ns < min_stages) return false;
  pl->nstages = ns;
  pl->nchains = p.D * p.B * p.C;
  // L2 priorities (experiments: GSPN_POL="x,vin,hin,vout,hout,acc", each 0|1|2)
  static const int def_pol[6] = {1, 0, 2, 0, 1, 1};
  for (int i = 0; i < 6; ++i) pl->pol[i] = def_pol[i];
  if (const char* e = getenv("GSPN_POL")) {
    int v[6], n = sscanf(e, "%d,%d,%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3], &v[4], &v[5]);
    for (int i = 0; i < n && i < 6; ++i) pl->pol[i] = v[i];
  }
  pl->smem_bytes = 1024 + ns * pl->stage_bytes + kSmemTail;
  pl->pair = ns >= 3 ? 1 : 0;
  if (const char* e = getenv("GSPN_PAIR")) pl->pair = pl->pair && atoi(e) != 0;
  if (const char* e = getenv("GSPN_NULL")) pl->null_compute = atoi(e) != 0;
  if (const char* e = getenv("GSPN_NOSLEEP")) pl->nosleep = atoi(e) != 0;
  return true;
}

bool fill_maps(StreamArgs* A, const void* const* ins, int nin, void* const* outs, const int64_t* in_planes,
               const int64_t* out_planes, int nout, gspn_dtype_t dt) {
  const Plan& pl = A->plan;
  const ScanParams& p = A->p;
  for (int t = 0; t < nin; ++t) {
    if (!encode(&A->in[0][t], ins[t], dt, p.W, p.H, in_planes[t], pl.bw, pl.K, CU_TENSOR_MAP_L2_PROMOTION_NONE))
      return false;
    const bool wide = pl.h_wide && t == nin - 1;  // bwd h_{t-1} view: 2K-step rows, 32-byte swizzle
    if (!encode(&A->in[1][t], ins[t], dt, p.W, p.H, in_planes[t], wide ? 2 * pl.K : pl.K, pl.bh, horiz_promotion(),
                wide))
      return false;
  }
  for (int t = 0; t < nout; ++t) {
    if (!encode(&A->out[0][t], outs[t], dt, p.W, p.H, out_planes[t], pl.bw, pl.K, CU_TENSOR_MAP_L2_PROMOTION_NONE))
      return false;
    if (!encode(&A->out[1][t], outs[t], dt, p.W, p.H, out_planes[t], pl.K, pl.bh, CU_TENSOR_MAP_L2_PROMOTION_NONE))
      return false;
  }
  return true;
}

template <typename KernelT>
cudaError_t launch(KernelT kernel, const StreamArgs& A, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(A.plan.smem_bytes));
  if (e != cudaSuccess) return e;
  const int threads = (A.plan.nwc + 2) * 32;  // consumers + producer + storer
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, A.plan.smem_bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = static_cast<int64_t>(sm_count()) * per_sm;
  if (const char* e = getenv("GSPN_GRID")) {  // experiments only: cap the persistent grid
    const int64_t g = atoll(e);
    if (g > 0 && g < grid) grid = g;
  }
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
  if (!make_plan(p, dt, F_NIN, 1, 2, /*two_ctas=*/true, /*E=*/4, &A.plan)) return cudaSuccess;
  const void* ins[F_NIN] = {p.x, p.lam, p.wl, p.wm, p.wr};
  const int64_t in_planes[F_NIN] = {p.B * p.C, p.D * p.B * p.C, p.D * p.B * p.G, p.D * p.B * p.G, p.D * p.B * p.G};
  void* outs[1] = {p.hout};
  const int64_t out_planes[1] = {p.D * p.B * p.C};
  if (!fill_maps(&A, ins, F_NIN, outs, in_planes, out_planes, 1, dt)) return cudaSuccess;
  *handled = true;
  cudaError_t e;
  if (A.plan.nwc <= 6)
    e = dt == GSPN_BF16 ? launch(fwd_stream_kernel<__nv_bfloat16, 4, 6>, A, s) : launch(fwd_stream_kernel<float, 4, 6>, A, s);
  else
    e = dt == GSPN_BF16 ? launch(fwd_stream_kernel<__nv_bfloat16, 4, kEdgeW>, A, s)
                        : launch(fwd_stream_kernel<float, 4, kEdgeW>, A, s);
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
  // Positions per lane: 2 (more warps per chain, better latency hiding) while a chain fits in
  // kBwdE2Warps warps, else 4. GSPN_BWD_E=2|4 overrides (experiments).
  int E = 2;
  if (const char* ev = getenv("GSPN_BWD_E")) E = atoi(ev) == 4 ? 4 : 2;
  if (!make_plan(p, dt, B_NIN, nout, 2, /*two_ctas=*/false, E, &A.plan) || (E == 2 && A.plan.nwc > kBwdE2Warps)) {
    E = 4;
    if (!make_plan(p, dt, B_NIN, nout, 2, /*two_ctas=*/false, E, &A.plan)) return cudaSuccess;
  }
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
  using BF = __nv_bfloat16;
  if (dt == GSPN_BF16) {
    if (E == 2)
      e = grouped ? launch(bwd_stream_kernel<BF, 2, true, kBwdE2Warps>, A, s)
                  : launch(bwd_stream_kernel<BF, 2, false, kBwdE2Warps>, A, s);
    else
      e = grouped ? launch(bwd_stream_kernel<BF, 4, true, kEdgeW>, A, s) : launch(bwd_stream_kernel<BF, 4, false, kEdgeW>, A, s);
  } else {
    if (E == 2)
      e = grouped ? launch(bwd_stream_kernel<float, 2, true, kBwdE2Warps>, A, s)
                  : launch(bwd_stream_kernel<float, 2, false, kBwdE2Warps>, A, s);
    else
      e = grouped ? launch(bwd_stream_kernel<float, 4, true, kEdgeW>, A, s)
                  : launch(bwd_stream_kernel<float, 4, false, kEdgeW>, A, s);
  }
  *launches += 1;
  return e;
}

}  // namespace gspn
