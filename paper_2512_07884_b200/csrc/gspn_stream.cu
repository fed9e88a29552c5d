// gspn_stream.cu — the TMA-streaming fast path for sm_100a (B200). DESIGN.md §6 has the measured
// numbers behind each choice below.
//
// Forward: one persistent launch covers every requested direction ("Kernel Fuse";
// the paper's one-stream-per-direction concurrency, becomes a direction dimension of the
// work queue). Backward: one persistent launch for the adjoint recurrence (writes g, the adjoint
// state, to workspace) plus one TMA-staged launch for the outputs (dlam, dx, dw), which are
// elementwise in g, h, x, lam and w.
//
// Work item = one chain (direction k, batch b, channel c): a P-wide state marching L steps -- or a
// pack of npack chains side by side (small planes), or, for P > 512, a slice of a chain held by one
// CTA of a thread-block cluster. A CTA owns one work item at a time:
//  * warp NWC (producer) streams K-step tiles of every input tensor into a shared-memory ring with
//    TMA (cp.async.bulk.tensor.3d + mbarrier complete_tx). K * sizeof(T) = 32 bytes: a horizontal
//    tile reads one full 32-byte DRAM sector of every row (narrower chunks measured at half the TMA
//    rate -- tools/tma_probe.cu, profiles/r1_notes.md);
//  * NWC consumer warps run the recurrence with the carry in fp32 registers. A warp covers 64
//    consecutive positions (2 per lane): it owns the middle 64 - 2 GH and recomputes GH ghost
//    positions on each side (temporal blocking), so neighbours move by warp shuffles every step and
//    warps exchange edge values through shared memory once per GH = K/2 steps (across the CTAs of a
//    cluster through distributed shared memory);
//  * warp NWC+1 (storer) writes horizontal tiles' outputs with TMA stores once the consumers have
//    written them in place over the consumed input rows; vertical chains store straight from
//    registers (a warp's owned positions are contiguous, so these stores coalesce).
// Lane mappings (both conflict-free on the shared-memory tiles):
//   T2B/B2T (vertical):   tile = K image rows x 512 positions ([box][K][512 B], packed: [K][npack][W]);
//                         a lane reads one 2-element vector per tensor per step.
//   L2R/R2L (horizontal): tile = up to 512 image rows x 32 bytes (TMA SWIZZLE_32B: 16-byte chunk ^=
//                         row bit 2); a lane owns 2 interleaved rows and reads each half-tile (K/2
//                         steps) of a row as one 16-byte vector.
// Work items are ordered (b, c)-major with the D directions adjacent and rotated per grid round, so
// co-scheduled CTAs share a plane's x through L2 and every CTA mixes vertical and horizontal chains.
//
// Backward recurrence: tiles in reverse step order; the carried state is
// (a g, b g, c g) of the previous step, so g_t = dh_t + (b g)[r] + (a g)[r+1] + (c g)[r-1]. The output
// kernels (a7) form dlam = g x, dx = sum_k g lam, and Da = g h_{t-1}[r-1], Db = g h_{t-1}[r],
// Dc = g h_{t-1}[r+1] summed over the group's channels, then apply the normalisation Jacobian.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>

#include "gspn_common.cuh"
#include "gspn_internal.h"
#include "gspn_ptx.cuh"

namespace gspn {
namespace {

using namespace ptx;

// Experiment knobs (A/B tooling under tools/): read only when GSPN_EXPERIMENTS is set, so a stray
// environment variable can never change what the product path computes or how it is scheduled.
const char* knob(const char* name) {
  static const bool on = getenv("GSPN_EXPERIMENTS") != nullptr;
  return on ? getenv(name) : nullptr;
}

constexpr int kMaxIn = 6;
constexpr int kMaxOut = 4;
constexpr int kEdgeW = 16;     // edge-buffer slots (>= consumer warps + 1)
// Fixed tile geometry (chains with P <= kPpad): one tensor's tile holds K steps x kPpad positions =
// 32 kPpad bytes; vertical tiles are [box][K][kRowB bytes] (box = kRowB / s positions), horizontal
// tiles [row][32 bytes]. Compile-time strides let every shared-memory read use an immediate offset.
constexpr int kPpad = 512;
constexpr uint32_t kTile = 32u * kPpad;
constexpr int kRowB = 512;
constexpr int kBarEdge = 1;    // named barrier ids (0 is __syncthreads)

template <typename T>
struct Cfg {
  static constexpr int es = static_cast<int>(sizeof(T));
  static constexpr int K = 32 / es;   // steps per tile (one 32-byte row of a horizontal tile)
  static constexpr int KS = K / 2;    // steps per half-tile (one 16-byte chunk)
  static constexpr int GH = KS;       // ghost positions on each side of a warp (exchange per half)
};

struct Plan {
  int K;               // steps per tile
  int E;               // positions per lane
  int own;             // positions a warp owns: 32 E - 2 GH
  int nwc;             // consumer warps
  int ppad;            // positions held by a tile (>= P, multiple of 64 and of bw)
  int es;              // element size in bytes
  int bw, nbw;         // vertical TMA box width (positions) and box count
  int bh, nbh;         // horizontal TMA box height (rows) and box count
  int nin;             // input tensors per tile
  // chain packing (G = C, max(H, W) <= kPpad / 2): npack chains of one direction side by side in a
  // tile, positions c * psub + r; vertical packed tiles are [K][npack][W] (one 3D box), horizontal
  // [npack][H][32 B]. Unpacked: npack = 1, vertical tiles [box][K][kRowB].
  int npack;
  int64_t nbc;         // B * C planes
  uint32_t vstep;      // bytes between consecutive steps of a vertical tile (kRowB, or npack W s)
  // P-split (P > one tile): a cluster of cl CTAs runs one chain, CTA s holds positions
  // [s ownc - GH, s ownc - GH + kPpad) and owns [s ownc, (s+1) ownc); slice-edge ghosts travel
  // through distributed shared memory. cl = 1: no cluster.
  int cl, ownc;
  int bhs, nbhs;       // cluster mode: horizontal TMA store boxes over the owned rows
  int nstages;
  uint32_t tile_bytes;   // one tensor's tile: K * ppad * es (= 32 * ppad)
  uint32_t stage_bytes;  // nin * tile_bytes
  uint32_t tx_v, tx_h;   // TMA bytes landing per stage (vertical / horizontal chains)
  int64_t nchains;
  uint32_t smem_bytes;
  // L2 eviction priority per access class (0 evict_first, 1 evict_normal, 2 evict_last):
  // x loads, vertical loads, horizontal loads, vertical stores, horizontal stores, fp32 accumulators
  int pol[6];
  int null_compute;    // experiments only (GSPN_NULL=1): consumers skip the arithmetic
  int fuse_h;          // fused backward: horizontal chains also form dw in the recurrence (else g only)
  int no_h;            // forward with checkpoints only (gspn_fwd_ckpt with h = NULL): h is not stored
  int nseg, kt;        // GSPN-local segment items: segments per chain slot, tiles per segment (nseg = 1: off)
  int hcp;             // forward: horizontal tap tiles by cp.async (producer_loop kHcp); full barriers count 33
  uint32_t tx_hc;      // TMA bytes of a horizontal stage when its tap tiles come by cp.async
};

struct alignas(64) StreamArgs {
  CUtensorMap in[2][kMaxIn];    // [0 vertical | 1 horizontal][tensor]
  CUtensorMap out[2][kMaxOut];
  ScanParams p;
  Plan plan;
  void* g;                      // bwd: adjoint state g [D,B,C,H,W] (I/O dtype, workspace)
  unsigned* ready;              // single-launch bwd: per (pack of) plane(s), chains whose g is complete
};

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------------------------ element access

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// E consecutive outputs from registers straight to global memory.
template <typename T, int E> struct GStore;
template <> struct GStore<__nv_bfloat16, 2> {
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float (&v)[2], uint64_t pol) {
    st_global_b32(p, pack_bf16x2(v[0], v[1]), pol);
  }
  static __device__ __forceinline__ void st_if(bool pred, __nv_bfloat16* p, const float (&v)[2], uint64_t pol) {
#ifdef GSPN_STORE_HINT
    st_global_b32_if(pred, p, pack_bf16x2(v[0], v[1]), pol);
#else
    (void)pol;
    st_global_cs_b32_if(pred, p, pack_bf16x2(v[0], v[1]));
#endif
  }
};
template <> struct GStore<float, 2> {
  static __device__ __forceinline__ void st(float* p, const float (&v)[2], uint64_t pol) {
    st_global_v2(p, __float_as_uint(v[0]), __float_as_uint(v[1]), pol);
  }
  static __device__ __forceinline__ void st_if(bool pred, float* p, const float (&v)[2], uint64_t pol) {
#ifdef GSPN_STORE_HINT
    st_global_v2_if(pred, p, __float_as_uint(v[0]), __float_as_uint(v[1]), pol);
#else
    (void)pol;
    st_global_cs_v2_if(pred, p, __float_as_uint(v[0]), __float_as_uint(v[1]));
#endif
  }
};

// One 16-byte chunk = KS steps of one row (horizontal tiles). Element indices are compile-time
// constants after unrolling, so the selects fold away.
template <typename T> struct Pk;
template <> struct Pk<__nv_bfloat16> {
  static __device__ __forceinline__ float get(const uint4& u, int i) {
    const uint32_t w = (i >> 1) == 0 ? u.x : (i >> 1) == 1 ? u.y : (i >> 1) == 2 ? u.z : u.w;
    return (i & 1) ? __uint_as_float(w & 0xFFFF0000u) : __uint_as_float(w << 16);
  }
  static __device__ __forceinline__ uint4 pack(const float (&v)[8]) {
    return make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                      pack_bf16x2(v[6], v[7]));
  }
};
template <> struct Pk<float> {
  static __device__ __forceinline__ float get(const uint4& u, int i) {
    return __uint_as_float(i == 0 ? u.x : i == 1 ? u.y : i == 2 ? u.z : u.w);
  }
  static __device__ __forceinline__ uint4 pack(const float (&v)[4]) {
    return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3]));
  }
};

// ------------------------------------------------------------------------------ chain bookkeeping

struct Chain {
  int k;            // direction slab
  bool vert, rev;   // orientation; reversed step order in canonical coordinates (B2T, R2L)
  int64_t bc, chain, wplane;  // first plane of the (pack of) chain(s): x, lam/h/dh, w
  int L, P, ntiles;
  int psub, nvalid;           // positions per chain; chains of the pack that exist
  int j0, j1;                 // scan-order tiles of this work item: [j0, j1) (a GSPN-local segment, or all)
};

// Work items are handed out round-robin over the persistent grid (CTAs, or clusters in P-split mode).
// kCl: P-split kernels (launched in clusters); the plain kernels carry none of the cluster logic.
template <bool kCl>
__device__ __forceinline__ int64_t work_first(const Plan&) {
  if constexpr (kCl) return static_cast<int64_t>(cluster_id_x());
  else return static_cast<int64_t>(blockIdx.x);
}
template <bool kCl>
__device__ __forceinline__ int64_t work_stride(const Plan&) {
  if constexpr (kCl) return static_cast<int64_t>(nclusters_x());
  else return static_cast<int64_t>(gridDim.x);
}
// First tile position held by this CTA (P-split: slice start minus the left ghosts).
template <bool kCl>
__device__ __forceinline__ int tile_base(const Plan& pl) {
  if constexpr (kCl) return static_cast<int>(cluster_ctarank()) * pl.ownc - pl.K / 2;
  else return 0;
}

// 64-bit index arithmetic: the backward kernels keep this form (with the 32-bit one below the config-4
// backward measured 1.5 % slower, 3 same-box reps, although its forward gained 3 %).
template <bool kCl>
__device__ __forceinline__ Chain make_chain64(const ScanParams& p, const Plan& pl, int64_t wi) {
  Chain ch;
  // GSPN-local segments as work items (the GSPN-2 grid over (chunk, n, c)): item wi is
  // segment wi % nseg of chain slot wi / nseg (nseg = 1: one item per chain)
  const int64_t w = wi / pl.nseg;
  const int seg = static_cast<int>(wi - w * pl.nseg);
  const int64_t bc = (w / p.D) * pl.npack;
  // Round i of the persistent grid covers slots [i G, (i+1) G): whole planes when D divides G. The
  // direction is rotated by i so every CTA cycles through all D directions (vertical and horizontal
  // chains run at different speeds; a fixed direction per CTA would leave the fast ones idle).
  const int64_t G = work_stride<kCl>(pl);
  ch.k = static_cast<int>(pl.nseg == 1 && G % p.D == 0 ? (w + w / G) % p.D : w % p.D);
  const uint32_t dir = p.dirbit[ch.k];
  ch.vert = (dir == GSPN_DIR_T2B) || (dir == GSPN_DIR_B2T);
  ch.rev = (dir == GSPN_DIR_B2T) || (dir == GSPN_DIR_R2L);
  ch.bc = bc;
  const int64_t b = bc / p.C, c = bc % p.C, g = c / (p.C / p.G);
  ch.chain = (ch.k * p.B + b) * p.C + c;
  ch.wplane = (ch.k * p.B + b) * p.G + g;
  ch.L = static_cast<int>(ch.vert ? p.H : p.W);
  ch.psub = static_cast<int>(ch.vert ? p.W : p.H);
  ch.P = ch.psub * pl.npack;
  ch.nvalid = static_cast<int>(pl.nbc - bc < pl.npack ? pl.nbc - bc : pl.npack);
  ch.ntiles = (ch.L + pl.K - 1) / pl.K;
  ch.j0 = 0;
  ch.j1 = ch.ntiles;
  if (pl.nseg > 1) {  // canonical tiles [c0, c1) of segment seg; reversed directions walk them backwards
    const int c0 = min(seg * pl.kt, ch.ntiles), c1 = min((seg + 1) * pl.kt, ch.ntiles);
    ch.j0 = ch.rev ? ch.ntiles - c1 : c0;
    ch.j1 = ch.rev ? ch.ntiles - c0 : c1;
  }
  return ch;
}

template <bool kCl>
__device__ __forceinline__ Chain make_chain32(const ScanParams& p, const Plan& pl, int64_t wi) {
  Chain ch;
  // GSPN-local segments as work items (the GSPN-2 grid over (chunk, n, c)): item wi is
  // segment wi % nseg of chain slot wi / nseg (nseg = 1: one item per chain). Every index here is < 2^31
  // (make_plan checks), so the divisions are 32-bit: a 64-bit division costs ~60 instructions, and every
  // warp of a CTA runs this once per work item (16 % of config 2's forward instructions when 64-bit).
  const uint32_t uw = static_cast<uint32_t>(wi);
  const uint32_t nseg = static_cast<uint32_t>(pl.nseg);
  const uint32_t w = nseg == 1 ? uw : uw / nseg;
  const int seg = static_cast<int>(uw - w * nseg);
  const uint32_t D = static_cast<uint32_t>(p.D);
  const uint32_t bcu = (w / D) * static_cast<uint32_t>(pl.npack);
  const int64_t bc = bcu;
  // Round i of the persistent grid covers slots [i G, (i+1) G): whole planes when D divides G. The
  // direction is rotated by i so every CTA cycles through all D directions (vertical and horizontal
  // chains run at different speeds; a fixed direction per CTA would leave the fast ones idle).
  const uint32_t G = static_cast<uint32_t>(work_stride<kCl>(pl));
  ch.k = static_cast<int>(nseg == 1 && G % D == 0 ? (w + w / G) % D : w % D);
  const uint32_t dir = p.dirbit[ch.k];
  ch.vert = (dir == GSPN_DIR_T2B) || (dir == GSPN_DIR_B2T);
  ch.rev = (dir == GSPN_DIR_B2T) || (dir == GSPN_DIR_R2L);
  ch.bc = bc;
  const uint32_t Cu = static_cast<uint32_t>(p.C);
  const uint32_t bu = bcu / Cu, cu = bcu - bu * Cu, gu = cu / (Cu / static_cast<uint32_t>(p.G));
  ch.chain = (static_cast<int64_t>(ch.k) * p.B + bu) * p.C + cu;
  ch.wplane = (static_cast<int64_t>(ch.k) * p.B + bu) * p.G + gu;
  ch.L = static_cast<int>(ch.vert ? p.H : p.W);
  ch.psub = static_cast<int>(ch.vert ? p.W : p.H);
  ch.P = ch.psub * pl.npack;
  ch.nvalid = static_cast<int>(pl.nbc - bc < pl.npack ? pl.nbc - bc : pl.npack);
  ch.ntiles = (ch.L + pl.K - 1) / pl.K;
  ch.j0 = 0;
  ch.j1 = ch.ntiles;
  if (pl.nseg > 1) {  // canonical tiles [c0, c1) of segment seg; reversed directions walk them backwards
    const int c0 = min(seg * pl.kt, ch.ntiles), c1 = min((seg + 1) * pl.kt, ch.ntiles);
    ch.j0 = ch.rev ? ch.ntiles - c1 : c0;
    ch.j1 = ch.rev ? ch.ntiles - c0 : c1;
  }
  return ch;
}

// Work item -> chain: the forward roles use the 32-bit form, the backward roles the 64-bit one (measured).
template <bool kCl, bool kFwd = false>
__device__ __forceinline__ Chain make_chain(const ScanParams& p, const Plan& pl, int64_t wi) {
  if constexpr (kFwd) return make_chain32<kCl>(p, pl, wi);
  else return make_chain64<kCl>(p, pl, wi);
}

// Canonical start coordinate (row for vertical, column for horizontal) of tile j (j counts tiles in
// scan order). Horizontal tiles sit on the K-aligned column grid (the 32-byte TMA swizzle needs an
// aligned inner coordinate), so for R2L with W % K != 0 the first tile is partial; vertical tiles
// just start K rows apart from the scan start.
__device__ __forceinline__ int tile_start(const Chain& ch, int j, int K) {
  if (!ch.rev) return j * K;
  return ch.vert ? (ch.L - (j + 1) * K) : (ch.ntiles - 1 - j) * K;
}

// A half-tile whose steps all lie outside [0, L) (the second half of a last partial tile, or for R2L the
// zero-filled columns past W of the first tile) changes nothing: skip its arithmetic (uniform across the
// CTA, so the edge exchange still runs). Vertical tiles start at the scan start; horizontal tiles sit on
// the K-aligned column grid, and for both L2R and R2L a half is outside iff its first column is >= W.
template <int K>
__device__ __forceinline__ bool half_outside_k(const Chain& ch, int j, int half, int cm) {
  if (ch.vert) return j * K + half * (K / 2) >= ch.L;
  return tile_start(ch, j, K) + cm * (K / 2) >= ch.L;
}

// Input tensor slots.
enum FwdIn { F_X = 0, F_LAM, F_WL, F_WM, F_WR, F_NIN };
enum BwdIn { B_DH = 0, B_WL, B_WM, B_WR, B_NIN };
// Fused backward (G = C): + h_{t-1} tiles. Vertical: B_H0 = the h rows one step earlier (box shifted by
// one row). Horizontal: B_H0 = h on the tile's own (K-aligned) columns, B_H1 = the neighbouring aligned
// tile on the side of step t-1 (its edge column is h_{t-1} of the tile's first step).
enum BwdFusedIn { B_H0 = B_NIN, B_H1, B_NINF };
// Merged backward (NEXT-1, hybrid path only): the B_DH slot holds the gate u, B_DY (= B_H1, unused by the
// hybrid) the upstream gradient dy of the direction merge; dh = s u dy is formed on the fly.
constexpr int B_DY = B_H1;

template <bool kBwd>
__device__ __forceinline__ int64_t plane_of(const Chain& ch, int slot) {
  const bool is_x = !kBwd && slot == F_X;
  const bool is_w = kBwd ? slot >= B_WL : slot >= F_WL;
  return is_x ? ch.bc : (is_w ? ch.wplane : ch.chain);
}

// ------------------------------------------------------------------------------ producer / storer

__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

// kHcp (forward, plain chains): the three tap tiles of a horizontal chain come through the LSU path
// (cp.async, 16 bytes per lane, all 32 lanes of the producer warp, completion on the stage's full barrier)
// instead of TMA, halving the TMA row requests of a horizontal stage (32-byte rows: request-rate bound).
template <bool kBwd, bool kCl, bool kXG = false, bool kHcp = false, bool k32 = !kBwd>
__device__ void producer_loop(const StreamArgs& A, uint8_t* ring, uint64_t* full, uint64_t* empty, int lane = 0) {
  const Plan& pl = A.plan;
  const uint64_t pol_xin = policy_of(pl.pol[0]);
  const uint64_t pol_vin = policy_of(pl.pol[1]);
  const uint64_t pol_hin = policy_of(pl.pol[2]);
  int stage = 0;
  uint32_t phase = 0;
  const int base = tile_base<kCl>(pl);
  for (int64_t w = work_first<kCl>(pl); w < pl.nchains; w += work_stride<kCl>(pl)) {
    const Chain ch = make_chain<kCl, k32>(A.p, pl, w);
    const int o = ch.vert ? 0 : 1;
    for (int jj = 0; jj < ch.j1 - ch.j0; ++jj) {
      const int j = kBwd ? (ch.j1 - 1 - jj) : (ch.j0 + jj);
      mbar_wait_sleep(smem_u32(&empty[stage]), phase ^ 1);
      const uint32_t fb = smem_u32(&full[stage]);
      const int s0 = tile_start(ch, j, pl.K);
      const uint32_t st = smem_u32(ring + static_cast<size_t>(stage) * pl.stage_bytes);
      if constexpr (kHcp) {
        if (!ch.vert) {  // tap tiles by cp.async: rows r = lane + 32 i, two 16-byte chunks each, 32-byte swizzle
          const int rows = pl.nbh * pl.bh;
          const int64_t HW = A.p.H * A.p.W;
          const void* tap[3] = {A.p.wl, A.p.wm, A.p.wr};
          for (int q = 0; q < 3; ++q) {
            const char* src0 = static_cast<const char*>(tap[q]) + (ch.wplane * HW + s0) * pl.es;
            const uint32_t dst0 = st + (F_WL + q) * pl.tile_bytes;
            for (int r = lane; r < rows; r += 32) {
              const bool in = base + r < A.p.H;
              const char* src = src0 + (in ? static_cast<int64_t>(base + r) * A.p.W * pl.es : 0);
              const uint32_t sw = static_cast<uint32_t>((r >> 2) & 1);
              cp_async16_zfill(dst0 + r * 32 + ((0u ^ sw) << 4), src, in ? 16u : 0u);
              cp_async16_zfill(dst0 + r * 32 + ((1u ^ sw) << 4), src + 16, in ? 16u : 0u);
            }
          }
        }
        cp_async_arrive_noinc(fb);  // every lane, every stage: the barrier counts 1 + 32 arrivals
        if (lane != 0) {
          if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
          continue;
        }
      }
      mbar_arrive_tx(fb, ch.vert ? pl.tx_v : (kHcp ? pl.tx_hc : pl.tx_h));
      for (int t = 0; t < pl.nin; ++t) {
        if (kHcp && !ch.vert && t >= F_WL) continue;
        const int tt = t + (kXG ? 1 : 0);  // kXG: the stage holds lam, w_l, w_m, w_r (x comes from L2)
        const int plane = static_cast<int>(plane_of<kBwd>(ch, tt));
        // x is re-read by the plane's other directions; vertical streams are read exactly once
        const uint64_t pol = (!kBwd && tt == F_X) ? pol_xin : (ch.vert ? pol_vin : pol_hin);
        const uint32_t dst = st + t * pl.tile_bytes;
        if (pl.npack > 1) {  // one 3D box: vertical (W, planes, rows), horizontal (cols, H, planes)
          if (ch.vert) tma_load3(dst, &A.in[0][t], 0, plane, s0, fb, pol);
          else tma_load3(dst, &A.in[1][t], s0, 0, plane, fb, pol);
        } else if (ch.vert) {
          for (int q = 0; q < pl.nbw; ++q)
            tma_load3(dst + q * pl.K * pl.bw * pl.es, &A.in[o][t], base + q * pl.bw, s0, plane, fb, pol);
        } else {
          for (int q = 0; q < pl.nbh; ++q)
            tma_load3(dst + q * pl.bh * 32, &A.in[o][t], s0, base + q * pl.bh, plane, fb, pol);
        }
      }
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
    }
  }
}

// Once the consumer warps of a horizontal tile have written its outputs in place (over consumed
// input rows) the storer sends them out with TMA, waits until the bulk copy has read shared memory,
// and only then hands the stage back to the producer. Vertical tiles store from registers, so their
// stage is released as soon as the consumers are done with it.
template <bool kCl, bool kFwdS = false>
__device__ void storer_loop(const StreamArgs& A, uint8_t* ring, uint64_t* done, uint64_t* empty, int nout,
                            const int* slots, bool bwd) {
  const Plan& pl = A.plan;
  const uint64_t pol = policy_of(pl.pol[4]);
  int stage = 0;
  uint32_t phase = 0;
  int64_t pending = -1;  // single-launch bwd: plane pack of the previous chain, published one chain later
  for (int64_t w = work_first<kCl>(pl); w < pl.nchains; w += work_stride<kCl>(pl)) {
    const Chain ch = make_chain<kCl, kFwdS>(A.p, pl, w);
    for (int jj = 0; jj < ch.j1 - ch.j0; ++jj) {
      const int j = bwd ? (ch.j1 - 1 - jj) : (ch.j0 + jj);
      mbar_wait_sleep(smem_u32(&done[stage]), phase);
      if (ch.vert && A.ready != nullptr) bulk_commit();  // an empty group: one group per tile either way
      if (!ch.vert) {
        const int s0 = tile_start(ch, j, pl.K);
        const uint8_t* st = ring + static_cast<size_t>(stage) * pl.stage_bytes;
        for (int t = 0; t < nout; ++t) {
          const uint32_t src = smem_u32(st + static_cast<size_t>(slots[t]) * pl.tile_bytes);
          if (pl.npack > 1) {
            tma_store3(&A.out[1][t], src, s0, 0, static_cast<int>(ch.chain), pol);
          } else if (kCl) {  // only the owned rows: the ghost rows belong to the neighbour CTAs
            const int gh = pl.K / 2;
            for (int q = 0; q < pl.nbhs; ++q)
              tma_store3(&A.out[1][t], src + (gh + q * pl.bhs) * 32, s0, tile_base<kCl>(pl) + gh + q * pl.bhs,
                         static_cast<int>(ch.chain), pol);
          } else {
            for (int q = 0; q < pl.nbh; ++q)
              tma_store3(&A.out[1][t], src + q * pl.bh * 32, s0, q * pl.bh, static_cast<int>(ch.chain), pol);
          }
        }
        bulk_commit();
        bulk_wait_read0();
      }
      mbar_arrive(smem_u32(&empty[stage]));
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
    }
    // Single-launch bwd: publish the PREVIOUS chain's plane once its stores are complete -- every bulk group
    // but this chain's last 8 (one per tile) -- so the storer never waits for its own latest stores.
    if (A.ready != nullptr) {
      if (pending >= 0) {
        if (ch.j1 - ch.j0 >= 8) bulk_wait_group8();
        else bulk_wait_all();
        fence_acq_rel_gpu();  // the consumers' g stores (observed through `done`) are gpu-visible
        fence_proxy_async_global();
        atomicAdd(A.ready + pending, 1u);
      }
      pending = ch.bc / pl.npack;
    }
  }
  bulk_wait_all();
  if (A.ready != nullptr && pending >= 0) {
    fence_acq_rel_gpu();
    fence_proxy_async_global();
    atomicAdd(A.ready + pending, 1u);
  }
}

// ------------------------------------------------------------------------------ per-lane geometry

// A warp covers 32 E = 64 consecutive positions starting at A = w * OWN - GH (OWN = 64 - 2 GH) and
// owns offsets [GH, 64 - GH); warp 0's left ghosts are the invalid positions -GH..-1. Vertical: lane
// holds positions A + 2 lane + e; horizontal: A + 32 q + lane (slot q), conflict-free on the tiles.
//
// Boundary handling without per-step masks: each lane gets byte-permute selectors (bf16) or
// and/or masks (fp32) that unpack its tap values already masked -- w_l -> 0 at r = 0, w_r -> 0 at
// r = P-1 (out-of-range taps, also dropped from S), and for positions outside [0, P) (TMA zero fill
// or clamped rows) w_l, w_r -> 0 and w_m -> 1, so those positions never couple into [0, P) -- in the
// forward through the masked taps of 0 and P-1, in the adjoint because their a g and c g are 0 --
// and stay finite. Steps outside [0, L) (partial first/last tiles) read TMA zero fill; the reciprocal is
// clamped so that S = 0 gives a zero update instead of 0 * inf.
constexpr int kE = 2;
constexpr int kMaxNWC = 11;                // consumer warps: 11 * 48 >= kPpad (bf16)
constexpr float kRcpMax = 1e30f;

__device__ __forceinline__ float bsel(uint32_t w, uint32_t sel) {
  return __uint_as_float(__byte_perm(w, 0x00003F80u, sel));  // bytes 4..7 = {0x80, 0x3F, 0, 0}
}
constexpr uint32_t kSelLo = 0x1066u, kSelHi = 0x3266u, kSelZero = 0x6666u, kSelOne = 0x5466u;

template <typename T>
struct Lanes {
  int A;
  bool own_v;            // vertical: both positions owned and < P
  bool own_h[kE];        // horizontal: slot owned and inside the tile
  uint32_t voff;         // vertical: byte offset of the lane's positions at kk = 0
  uint32_t hoff[kE];     // horizontal: slot row's byte offset, chunk 0 (chunk c: hoff ^ (c << 4))
  int64_t vout;          // vertical: element offset of the lane's first position in row 0 of its plane
  // tap unpack masks [tap l/m/r][element e | slot q][half / (and, or)]
  uint32_t s[3][kE][2];
  // forward with x read from global memory (kXG): element offsets of the lane's x in row / column 0
  int64_t xoff;          // vertical: the lane's 2 positions of plane row 0
  int64_t xho[kE];       // horizontal: start of each slot's row
  bool xv_ok, xh_ok[kE];
};

// r: tile position; psub: positions per chain; nvalid: chains present (packing). A chain's taps at its
// own first / last position are dropped, which also decouples packed neighbours.
template <typename T>
__device__ __forceinline__ void tap_masks(int r, int psub, int nvalid, uint32_t (&sl)[2], uint32_t (&sm)[2],
                                          uint32_t (&sr)[2], int half_for_bf16) {
  const bool valid = r >= 0 && r < psub * nvalid;
  const int rl = valid ? r % psub : 0;
  const bool kl = valid && rl >= 1, kr = valid && rl <= psub - 2;
  if constexpr (sizeof(T) == 2) {
    // half_for_bf16: -1 -> fill both halves (horizontal slot), 0/1 -> element in the low/high half
    for (int hh = 0; hh < 2; ++hh) {
      const int hf = half_for_bf16 < 0 ? hh : half_for_bf16;
      const uint32_t keep = hf ? kSelHi : kSelLo;
      sl[hh] = kl ? keep : kSelZero;
      sr[hh] = kr ? keep : kSelZero;
      sm[hh] = valid ? keep : kSelOne;
    }
  } else {
    sl[0] = kl ? 0xFFFFFFFFu : 0u; sl[1] = 0u;
    sr[0] = kr ? 0xFFFFFFFFu : 0u; sr[1] = 0u;
    sm[0] = valid ? 0xFFFFFFFFu : 0u; sm[1] = valid ? 0u : 0x3F800000u;
  }
}

template <typename T, bool kCl>
__device__ __forceinline__ Lanes<T> make_lanes(const Plan& pl, const ScanParams& p, const Chain& ch, int wi,
                                               int lane) {
  using C = Cfg<T>;
  constexpr int WARP = 32 * kE, OWN = WARP - 2 * C::GH;
  Lanes<T> ln;
  const int base = tile_base<kCl>(pl);  // tile row = position - base
  ln.A = (kCl ? base : -C::GH) + wi * OWN;
  constexpr int lo = C::GH;
  const int nval = ch.psub * ch.nvalid;
  // vertical
  {
    const int off = kE * lane;
    const int r0 = ln.A + off;
    ln.own_v = off >= lo && off < WARP - C::GH && r0 >= 0 && r0 < nval;
    const int rt = r0 - base;
    const int rc = rt < 0 ? 0 : (rt > kPpad - kE ? kPpad - kE : rt);
    if (pl.npack > 1) {
      ln.voff = static_cast<uint32_t>(rc * C::es);
    } else {
      const int bw = kRowB / C::es;
      ln.voff = static_cast<uint32_t>((rc / bw) * (C::K * kRowB) + (rc % bw) * C::es);
    }
    const int rv = r0 < 0 ? 0 : r0;
    ln.vout = (ch.chain + rv / ch.psub) * (p.H * p.W) + rv % ch.psub;  // P % kE == 0: both positions in one chain
    ln.xv_ok = r0 >= 0 && r0 < nval;
    ln.xoff = (ch.bc + rv / ch.psub) * (p.H * p.W) + rv % ch.psub;
  }
  // horizontal
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    const int off = 32 * q + lane;
    const int r = ln.A + off;
    const int rt = r - base;
    ln.own_h[q] = off >= lo && off < WARP - C::GH && rt < kPpad;  // rows >= P: outside the store box
    const uint32_t rc = static_cast<uint32_t>(rt < 0 ? 0 : (rt >= kPpad ? kPpad - 1 : rt));
    ln.hoff[q] = rc * 32 + (((rc >> 2) & 1u) << 4);
    ln.xh_ok[q] = r >= 0 && r < nval;
    const int rr = r < 0 ? 0 : r;
    ln.xho[q] = (ch.bc + rr / ch.psub) * (p.H * p.W) + static_cast<int64_t>(rr % ch.psub) * p.W;
  }
  if (ch.vert) {
#pragma unroll
    for (int e = 0; e < kE; ++e)
      tap_masks<T>(ln.A + kE * lane + e, ch.psub, ch.nvalid, ln.s[0][e], ln.s[1][e], ln.s[2][e], e);
  } else {
#pragma unroll
    for (int q = 0; q < kE; ++q)
      tap_masks<T>(ln.A + 32 * q + lane, ch.psub, ch.nvalid, ln.s[0][q], ln.s[1][q], ln.s[2][q], -1);
  }
  return ln;
}

// Vertical step operands: 2 consecutive positions per tensor from one 4- (bf16) or 8-byte (fp32) read.
template <typename T>
__device__ __forceinline__ void vload(const uint8_t* p, float (&v)[2]) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
    v[0] = __uint_as_float(u << 16);
    v[1] = __uint_as_float(u & 0xFFFF0000u);
  } else {
    const float2 u = *reinterpret_cast<const float2*>(p);
    v[0] = u.x; v[1] = u.y;
  }
}
template <typename T>
__device__ __forceinline__ void vload_tap(const uint8_t* p, const uint32_t (&m)[kE][2], float (&v)[2]) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
    v[0] = bsel(u, m[0][0]);
    v[1] = bsel(u, m[1][0]);
  } else {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    v[0] = __uint_as_float((u.x & m[0][0]) | m[0][1]);
    v[1] = __uint_as_float((u.y & m[1][0]) | m[1][1]);
  }
}

// Horizontal chunk element i (memory order) of a 16-byte vector; tap version applies the slot masks.
template <typename T>
__device__ __forceinline__ float hget(const uint4& u, int i) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t w = (i >> 1) == 0 ? u.x : (i >> 1) == 1 ? u.y : (i >> 1) == 2 ? u.z : u.w;
    return (i & 1) ? __uint_as_float(w & 0xFFFF0000u) : __uint_as_float(w << 16);
  } else {
    return __uint_as_float(i == 0 ? u.x : i == 1 ? u.y : i == 2 ? u.z : u.w);
  }
}
template <typename T>
__device__ __forceinline__ float hget_tap(const uint4& u, int i, const uint32_t (&m)[2]) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t w = (i >> 1) == 0 ? u.x : (i >> 1) == 1 ? u.y : (i >> 1) == 2 ? u.z : u.w;
    return bsel(w, m[i & 1]);
  } else {
    const uint32_t w = i == 0 ? u.x : i == 1 ? u.y : i == 2 ? u.z : u.w;
    return __uint_as_float((w & m[0]) | m[1]);
  }
}

// Ghost exchange through shared memory, without divergent branches: every lane stores all of its
// values into its warp's 64-slot row of the exchange buffer [array][par][warp][64]; after the named
// barrier every lane reads back one value per slot from a per-lane precomputed source -- a ghost
// slot from the neighbouring warp's owned edge (offset +-(64 - 2 GH)), any other slot from itself.
// Warp 0's left and the last warp's right ghosts keep their own (outside-the-chain) values.
constexpr int kXRow = 64;  // floats per warp row of the exchange buffer
constexpr int kXArr = 2 * kEdgeW * kXRow;  // floats per state array (2 parities)

struct XSrc {
  uint32_t v;      // vertical: byte offset (within one parity plane) of the lane's 2 source values
  uint32_t h[kE];  // horizontal: byte offset of each slot's source value
};

template <typename T>
__device__ __forceinline__ XSrc make_xsrc(int wi, int nwc, int lane) {
  using C = Cfg<T>;
  constexpr int WARP = 32 * kE, SH = WARP - 2 * C::GH;  // ghost <-> neighbour's owned edge distance
  XSrc x;
  {
    const int o = kE * lane;
    int sw = wi, so = o;
    if (o < C::GH && wi > 0) { sw = wi - 1; so = o + SH; }
    else if (o >= WARP - C::GH && wi < nwc - 1) { sw = wi + 1; so = o - SH; }
    x.v = static_cast<uint32_t>((sw * kXRow + so) * 4);
  }
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    const int o = 32 * q + lane;
    int sw = wi, so = o;
    if (o < C::GH && wi > 0) { sw = wi - 1; so = o + SH; }
    else if (o >= WARP - C::GH && wi < nwc - 1) { sw = wi + 1; so = o - SH; }
    x.h[q] = static_cast<uint32_t>((sw * kXRow + so) * 4);
  }
  return x;
}

// buf: exchange buffer of one state array at parity par.
__device__ __forceinline__ void edge_publish(float* buf, int wi, int lane, bool vert, const float (&v)[kE]) {
  float* row = buf + wi * kXRow;
  if (vert) {
    *reinterpret_cast<float2*>(row + kE * lane) = make_float2(v[0], v[1]);
  } else {
    row[lane] = v[0];
    row[32 + lane] = v[1];
  }
}

__device__ __forceinline__ void edge_reload(const float* buf, const XSrc& x, bool vert, float (&v)[kE]) {
  const char* b = reinterpret_cast<const char*>(buf);
  if (vert) {
    const float2 u = *reinterpret_cast<const float2*>(b + x.v);
    v[0] = u.x;
    v[1] = u.y;
  } else {
    v[0] = *reinterpret_cast<const float*>(b + x.h[0]);
    v[1] = *reinterpret_cast<const float*>(b + x.h[1]);
  }
}

// Shared-memory carve-up common to both kernels: ring | full | empty | done | edges | cluster edges.
struct Smem {
  uint8_t* ring;
  uint64_t *full, *empty, *done;
  float* edge;
  float *xl, *xr;   // P-split: ghost values from the left / right neighbour CTA [3 arrays][2 par][8]
  uint64_t* xb;     // P-split: [0..1] left-neighbour data landed (par), [2..3] right-neighbour data landed
};

__device__ __forceinline__ Smem carve(uint8_t* smem_raw, const Plan& pl) {
  Smem m;
  m.ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared space
  m.full = reinterpret_cast<uint64_t*>(m.ring + static_cast<size_t>(pl.nstages) * pl.stage_bytes);
  m.empty = m.full + pl.nstages;
  m.done = m.empty + pl.nstages;
  m.edge = reinterpret_cast<float*>(m.done + pl.nstages);  // [3 state arrays][2 par][kEdgeW][64]
  m.xl = m.edge + 3 * kXArr;
  m.xr = m.xl + 3 * 2 * 8;
  m.xb = reinterpret_cast<uint64_t*>(m.xr + 3 * 2 * 8);
  return m;
}

template <bool kCl>
__device__ __forceinline__ void init_barriers(const Smem& m, const Plan& pl) {
  // Packed tiles: zero the ring once; lanes may read tile rows past the packed chains that no TMA box
  // writes, and those rows must hold finite values (zero, or earlier tiles' data). Unpacked plans
  // size their boxes to cover every row a lane reads.
  if (pl.npack > 1) {
    uint4* r = reinterpret_cast<uint4*>(m.ring);
    const uint32_t n = pl.nstages * pl.stage_bytes / 16;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) r[i] = make_uint4(0u, 0u, 0u, 0u);
    fence_proxy_async();  // generic-proxy zeros ordered before the TMA (async-proxy) writes
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < pl.nstages; ++s) {
      mbar_init(smem_u32(&m.full[s]), pl.hcp ? 33 : 1);  // producer arrive + TMA bytes (+ 32 cp.async lanes)
      mbar_init(smem_u32(&m.empty[s]), 1);      // storer
      mbar_init(smem_u32(&m.done[s]), pl.nwc);  // one arrive per consumer warp
    }
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&m.xb[i]), 1);  // the receiver's arrive.expect_tx
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if constexpr (kCl) cluster_sync_all();  // neighbours' barriers initialised before any remote access
}

// ---- P-split ghost exchange between the CTAs of a cluster (after the intra-CTA publish).
// Warp 0 of CTA s sends its first GH owned values to CTA s-1 (they are that CTA's right ghosts), the
// last warp sends its last GH owned values to CTA s+1 with st.async, each store completing its bytes on
// the receiver's barrier, which the receiver arms per half (arrive.expect_tx). Parity-double-buffered like
// the local edges;
// a sender cannot run two halves ahead because it needs the receiver's edges of the half between.
// side 0: towards rank - 1, side 1: towards rank + 1.
__device__ __forceinline__ bool xgo(int side, int wi, int nwc, int rank, int cl) {
  return side == 0 ? (wi == 0 && rank > 0) : (wi == nwc - 1 && rank < cl - 1);
}

// st.async: the remote store itself signals the receiver's mbarrier (complete_tx) when the value has landed,
// so the sender needs no release fence -- a release at cluster scope would also wait for this thread's
// outstanding global stores (the h / g rows of the vertical chains) on every exchange.
template <typename T>
__device__ __forceinline__ void xput(const Smem& m, int par, int side, uint32_t tr, int a, int lane, bool vert,
                                     const float (&v)[kE]) {
  using C = Cfg<T>;
  constexpr int WARP = 32 * kE;
  float* dst = (side == 0 ? m.xr : m.xl) + (a * 2 + par) * 8;  // left-going data = receiver's right ghosts
  const uint32_t bar = mapa(smem_u32(&m.xb[(side == 0 ? 2 : 0) + par]), tr);
  if (vert) {
    const int o = kE * lane;
    const int lo = side == 0 ? C::GH : WARP - 2 * C::GH;
    if (o >= lo && o < lo + C::GH) {
#pragma unroll
      for (int e = 0; e < kE; ++e) st_async_f32(mapa(smem_u32(dst + o - lo + e), tr), v[e], bar);
    }
  } else {
    const int lo = side == 0 ? C::GH : 32 - 2 * C::GH;
    if (lane >= lo && lane < lo + C::GH)
      st_async_f32(mapa(smem_u32(dst + lane - lo), tr), side == 0 ? v[0] : v[kE - 1], bar);
  }
}

__device__ __forceinline__ void xarrive(const Smem&, int, int, uint32_t) {}

// The receiving warp arms its barrier for this half's bytes (GH values per exchanged array) and waits.
template <typename T>
__device__ __forceinline__ void xwait(const Smem& m, int par, int side, uint32_t xphase, int narr) {
  const uint32_t bar = smem_u32(&m.xb[(side == 0 ? 0 : 2) + par]);
  if ((threadIdx.x & 31) == 0) mbar_arrive_tx(bar, static_cast<uint32_t>(narr * Cfg<T>::GH * 4));
  mbar_wait_cluster(bar, xphase);
}

template <typename T>
__device__ __forceinline__ void xget(const Smem& m, int par, int side, int a, int lane, bool vert, float (&v)[kE]) {
  using C = Cfg<T>;
  constexpr int WARP = 32 * kE;
  const float* src = (side == 0 ? m.xl : m.xr) + (a * 2 + par) * 8;
  if (vert) {
    const int o = kE * lane;
    const int lo = side == 0 ? 0 : WARP - C::GH;
    if (o >= lo && o < lo + C::GH) {
#pragma unroll
      for (int e = 0; e < kE; ++e) v[e] = src[o - lo + e];
    }
  } else {
    const int lo = side == 0 ? 0 : 32 - C::GH;
    if (lane >= lo && lane < lo + C::GH) {
      if (side == 0) v[0] = src[lane - lo];
      else v[kE - 1] = src[lane - lo];
    }
  }
}

// Every thread of every role passes one final cluster barrier: no CTA leaves while a neighbour may
// still address its shared memory.
template <bool kCl>
__device__ __forceinline__ void cluster_exit() {
  __syncwarp();
  if constexpr (kCl) cluster_sync_all();
}

__device__ __forceinline__ float clamped_rcp(float s) { return fminf(fast_rcp(s), kRcpMax); }

// Normaliser modes (kernel template parameter): pre-normalised taps (1 / S = 1); raw taps with the
// clamped reciprocal (chains with partial tiles read zero-filled steps, S = 0); raw taps when every
// L is a multiple of K (no zero-filled steps: S > 0 at valid positions, S = 1 at masked ones).
enum NormMode { kNormPre = 0, kNormClamp = 1, kNormFull = 2 };
template <int kMode>
__device__ __forceinline__ float norm_inv(float s) {
  if constexpr (kMode == kNormPre) return 1.f;
  else if constexpr (kMode == kNormClamp) return clamped_rcp(s);
  else return fast_rcp(s);
}

// GSPN-local (R19): bit p of the result is set when the p-th step a half
// processes starts a kchunk segment in scan order. c_first: canonical scan-axis index (row / column) of
// that half's first processed step; cstep = +-1: canonical index change per processed step; scan_fwd:
// T2B / L2R (segment start s % k == 0) vs B2T / R2L ((s + 1) % k == 0). One modulo per half.
__device__ __forceinline__ uint32_t reset_bits(int c_first, int cstep, bool scan_fwd, int k, int n) {
  const int target = scan_fwd ? 0 : k - 1;  // residue of a segment's first scan step
  int o = (cstep * (target - c_first)) % k;
  if (o < 0) o += k;
  uint32_t m = 0;
  for (; o < n; o += k) m |= 1u << o;
  return m;
}

// ------------------------------------------------------------------------------ forward

// One step of Eq. 1 at one position (taps already masked, see Lanes).
template <int kPre>
__device__ __forceinline__ float fwd_math(float x, float lam, float l, float m, float r, float hm1, float h,
                                          float hp1) {
  const float acc = fmaf(l, hm1, fmaf(m, h, r * hp1));
  const float inv = norm_inv<kPre>((l + r) + m);
  return fmaf(acc, inv, lam * x);
}

// x of one half-tile held in registers (forward with x read from global memory, kXG): x is shared by the
// D directions of a plane, so it is mostly served by L2; leaving it out of the TMA stage frees a ring slot
// (4 tiles per stage instead of 5: 3 stages instead of 2). Loaded one half ahead of its use.
template <typename T>
struct XPre {
  static constexpr int kV = Cfg<T>::KS * static_cast<int>(sizeof(T)) / 2;  // vertical: 2 elements per step
  uint32_t v[kV];
  uint4 h[kE];  // horizontal: the KS-step chunk of each slot's row
};

template <typename T>
__device__ __forceinline__ void x_fetch(XPre<T>& xp, const Lanes<T>& ln, const Chain& ch, const T* xg, int j, int half,
                                        int64_t W) {
  using C = Cfg<T>;
  if (ch.vert) {
    const int t0 = j * C::K + half * C::KS;
#pragma unroll
    for (int ss = 0; ss < C::KS; ++ss) {
      const int t = t0 + ss;
      const bool ok = ln.xv_ok && t < ch.L;
      const int row = ch.rev ? ch.L - 1 - t : t;
      const T* a = xg + ln.xoff + static_cast<int64_t>(ok ? row : 0) * W;
      if constexpr (sizeof(T) == 2) {
        xp.v[ss] = ok ? __ldg(reinterpret_cast<const unsigned int*>(a)) : 0u;
      } else {
        const uint2 u = ok ? __ldg(reinterpret_cast<const uint2*>(a)) : make_uint2(0u, 0u);
        xp.v[2 * ss] = u.x;
        xp.v[2 * ss + 1] = u.y;
      }
    }
  } else {
    const int cm = ch.rev ? 1 - half : half;
    const int64_t c0 = tile_start(ch, j, C::K) + cm * C::KS;
#pragma unroll
    for (int q = 0; q < kE; ++q)
      xp.h[q] = ln.xh_ok[q] ? ld_nc_v4(xg + ln.xho[q] + c0) : make_uint4(0u, 0u, 0u, 0u);
  }
}

// Vertical half-tile: KS steps; p0 = the lane's operands at the half's first step, stepb = +-kRowB.
// New states go straight to global memory (gp advances by gstep rows per step).
template <typename T, int kPre, bool kLocal, bool kXG = false>
__device__ __forceinline__ void fwd_half_vert(const Lanes<T>& ln, const uint8_t* p0, int stepb, T* gp,
                                              int64_t gstep, int t0, int L, float (&h)[kE], uint64_t pol,
                                              uint32_t rm, const XPre<T>* xp = nullptr) {
  constexpr int KS = Cfg<T>::KS;
  constexpr int o = kXG ? 1 : 0;  // kXG: x is not in the stage, the other tiles move down one slot
  // store predicate and pointer stepping hoisted out of the step loop (the null check is taken once)
  const bool on = ln.own_v && gp != nullptr;
  const int nv = L - t0;  // steps of this half inside [0, L)
  uintptr_t ga = reinterpret_cast<uintptr_t>(gp);
  const intptr_t gsb = static_cast<intptr_t>(gstep) * static_cast<intptr_t>(sizeof(T));
#pragma unroll
  for (int ss = 0; ss < KS; ++ss) {
    if constexpr (kLocal) {  // segment start: h_{t-1} does not propagate (warp-uniform)
      if ((rm >> ss) & 1u) h[0] = h[1] = 0.f;
    }
    const uint8_t* q = p0 + ss * stepb;
    float x[2], lam[2], l[2], m[2], r[2];
    if constexpr (kXG) {
      if constexpr (sizeof(T) == 2) {
        x[0] = __uint_as_float(xp->v[ss] << 16);
        x[1] = __uint_as_float(xp->v[ss] & 0xFFFF0000u);
      } else {
        x[0] = __uint_as_float(xp->v[2 * ss]);
        x[1] = __uint_as_float(xp->v[2 * ss + 1]);
      }
    } else {
      vload<T>(q + F_X * kTile, x);
    }
    vload<T>(q + (F_LAM - o) * kTile, lam);
    vload_tap<T>(q + (F_WL - o) * kTile, ln.s[0], l);
    vload_tap<T>(q + (F_WM - o) * kTile, ln.s[1], m);
    vload_tap<T>(q + (F_WR - o) * kTile, ln.s[2], r);
    const float left = __shfl_up_sync(0xffffffffu, h[1], 1);    // lane 0: own value (ghost or masked)
    const float right = __shfl_down_sync(0xffffffffu, h[0], 1);  // lane 31: own value
    const float h0 = fwd_math<kPre>(x[0], lam[0], l[0], m[0], r[0], left, h[0], h[1]);
    const float h1 = fwd_math<kPre>(x[1], lam[1], l[1], m[1], r[1], h[0], h[1], right);
    h[0] = h0;
    h[1] = h1;
    GStore<T, 2>::st_if(on && ss < nv, reinterpret_cast<T*>(ga), h, pol);
    ga += gsb;
  }
}

// Horizontal neighbours: position A + 32 q + lane; lane 0 of slot 1 takes lane 31 of slot 0 and
// lane 31 of slot 0 takes lane 0 of slot 1 (the warp's outermost positions are ghosts or masked).
__device__ __forceinline__ void slot_lo(const float (&v)[kE], int lane, float (&lo)[kE]) {
  const float u0 = __shfl_sync(0xffffffffu, v[0], (lane + 31) & 31);
  const float u1 = __shfl_sync(0xffffffffu, v[1], (lane + 31) & 31);
  lo[0] = u0;
  lo[1] = lane == 0 ? u0 : u1;
}
__device__ __forceinline__ void slot_hi(const float (&v)[kE], int lane, float (&hi)[kE]) {
  const float d0 = __shfl_sync(0xffffffffu, v[0], (lane + 1) & 31);
  const float d1 = __shfl_sync(0xffffffffu, v[1], (lane + 1) & 31);
  hi[0] = lane == 31 ? d1 : d0;
  hi[1] = d1;
}

// Horizontal half-tile: one 16-byte chunk (KS steps) per tensor per slot; kRev walks the chunk
// backwards (R2L). The new states come back packed in memory order for the in-place write.
template <typename T, int kPre, bool kRev, bool kLocal, bool kXG = false>
__device__ __forceinline__ void fwd_half_horiz(const Lanes<T>& ln, const uint8_t* st, int cm, int lane,
                                               float (&h)[kE], uint4 (&OUT)[kE], uint32_t rm,
                                               const XPre<T>* xp = nullptr) {
  constexpr int KS = Cfg<T>::KS;
  constexpr int o = kXG ? 1 : 0;
  uint4 X[kE], LAM[kE], WL[kE], WM[kE], WR[kE];
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    const uint32_t off = ln.hoff[q] ^ (static_cast<uint32_t>(cm) << 4);
    if constexpr (kXG) X[q] = xp->h[q];
    else X[q] = *reinterpret_cast<const uint4*>(st + F_X * kTile + off);
    LAM[q] = *reinterpret_cast<const uint4*>(st + (F_LAM - o) * kTile + off);
    WL[q] = *reinterpret_cast<const uint4*>(st + (F_WL - o) * kTile + off);
    WM[q] = *reinterpret_cast<const uint4*>(st + (F_WM - o) * kTile + off);
    WR[q] = *reinterpret_cast<const uint4*>(st + (F_WR - o) * kTile + off);
  }
  float O[kE][KS];
#pragma unroll
  for (int ss = 0; ss < KS; ++ss) {
    const int i = kRev ? KS - 1 - ss : ss;  // element of the chunk (memory order)
    if constexpr (kLocal) {
      if ((rm >> ss) & 1u) h[0] = h[1] = 0.f;
    }
    float lo[kE], hi[kE];
    slot_lo(h, lane, lo);
    slot_hi(h, lane, hi);
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      h[q] = fwd_math<kPre>(hget<T>(X[q], i), hget<T>(LAM[q], i), hget_tap<T>(WL[q], i, ln.s[0][q]),
                            hget_tap<T>(WM[q], i, ln.s[1][q]), hget_tap<T>(WR[q], i, ln.s[2][q]), lo[q], h[q], hi[q]);
      O[q][i] = h[q];
    }
  }
#pragma unroll
  for (int q = 0; q < kE; ++q) OUT[q] = Pk<T>::pack(O[q]);
}

// Body of the forward scan (every role returns from here when its work is done); the barriers of `m` must
// be initialised. Shared by fwd_stream_kernel and the merged single launch fwd_one_kernel.
template <typename T, int kPre, bool kCl, bool kLocal, bool kXG = false>
__device__ __forceinline__ void fwd_stream_body(const StreamArgs& A, const Smem& m) {
  using C = Cfg<T>;
  const Plan& pl = A.plan;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kOutSlot = kXG ? 0 : F_X;  // in-place horizontal outputs: over the x (or, kXG, lam) chunk
  if (warp == pl.nwc) {  // producer warp
    if (lane == 0)
      for (int o = 0; o < 2; ++o)
        for (int t = 0; t < pl.nin; ++t) asm volatile("prefetch.tensormap [%0];" ::"l"(&A.in[o][t]) : "memory");
    if constexpr (!kCl && !kXG) {
      if (pl.hcp) producer_loop<false, false, false, true>(A, m.ring, m.full, m.empty, lane);
      else if (lane == 0) producer_loop<false, kCl, kXG>(A, m.ring, m.full, m.empty);
    } else if (lane == 0) {
      producer_loop<false, kCl, kXG>(A, m.ring, m.full, m.empty);
    }
    cluster_exit<kCl>();
    return;
  }
  if (warp == pl.nwc + 1) {  // storer warp
    if (lane == 0) {
      const int slots[1] = {kOutSlot};
      storer_loop<kCl, true>(A, m.ring, m.done, m.empty, pl.no_h ? 0 : 1, slots, false);
    }
    cluster_exit<kCl>();
    return;
  }
  const uint64_t pol_vout = policy_of(pl.pol[3]);
  const int nthreads = pl.nwc * 32;
  const int64_t W = A.p.W;
  const int kchunk = static_cast<int>(A.p.kchunk);
  const int rank = kCl ? static_cast<int>(cluster_ctarank()) : 0;
  const XSrc xs = make_xsrc<T>(warp, pl.nwc, lane);
  uint32_t xphase = 0;  // P-split: phase bit of the cluster edge barriers, per parity
  int stage = 0, par = 0;
  uint32_t phase = 0;
  const T* const xg = static_cast<const T*>(A.p.x);
  float* const ckpt = A.p.ckpt;                           // NEXT-3 checkpoints (unpacked, unsplit chains)
  const int64_t ckstride = A.p.H * A.p.W / C::KS;        // floats per chain
  for (int64_t w = work_first<kCl>(pl); w < pl.nchains; w += work_stride<kCl>(pl)) {
    const Chain ch = make_chain<kCl, true>(A.p, pl, w);
    const Lanes<T> ln = make_lanes<T, kCl>(pl, A.p, ch, warp, lane);
    T* hout = pl.no_h ? nullptr : static_cast<T*>(A.p.hout) + ln.vout;
    float h[kE] = {0.f, 0.f};
    XPre<T> xcur;
    if constexpr (kXG) x_fetch<T>(xcur, ln, ch, xg, ch.j0, 0, W);
    for (int j = ch.j0; j < ch.j1; ++j) {
      mbar_wait_sleep(smem_u32(&m.full[stage]), phase);
      __syncwarp();  // reconverge after the per-thread spin: the shuffles below need no collective fallback
      uint8_t* st = m.ring + static_cast<size_t>(stage) * pl.stage_bytes;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        uint4 OUT[kE];
        const int cm = ch.rev ? 1 - half : half;  // horizontal: memory chunk of this half
        const bool live = !pl.null_compute && !half_outside_k<C::K>(ch, j, half, cm);
        XPre<T> xnext;
        if constexpr (kXG) {  // the next half's x, loaded while this half computes
          const int jn = half == 0 ? j : j + 1, hn = half ^ 1;
          if (jn < ch.j1) x_fetch<T>(xnext, ln, ch, xg, jn, hn, W);
        }
        if (live) {
          uint32_t rm = 0;
          if (ch.vert) {
            const int t0 = j * C::K + half * C::KS;
            const int kk0 = ch.rev ? C::K - 1 - half * C::KS : half * C::KS;
            const int row0 = ch.rev ? ch.L - 1 - t0 : t0;
            const int vs = static_cast<int>(pl.vstep);
            if constexpr (kLocal) rm = reset_bits(row0, ch.rev ? -1 : 1, !ch.rev, kchunk, C::KS);
            fwd_half_vert<T, kPre, kLocal, kXG>(ln, st + ln.voff + kk0 * vs, ch.rev ? -vs : vs,
                                                hout ? hout + static_cast<int64_t>(row0) * W : nullptr,
                                                ch.rev ? -W : W, t0, ch.L, h, pol_vout, rm, &xcur);
          } else {
            if constexpr (kLocal)
              rm = reset_bits(tile_start(ch, j, C::K) + cm * C::KS + (ch.rev ? C::KS - 1 : 0), ch.rev ? -1 : 1,
                              !ch.rev, kchunk, C::KS);
            if (ch.rev) fwd_half_horiz<T, kPre, true, kLocal, kXG>(ln, st, cm, lane, h, OUT, rm, &xcur);
            else fwd_half_horiz<T, kPre, false, kLocal, kXG>(ln, st, cm, lane, h, OUT, rm, &xcur);
          }
        }
        if constexpr (kXG) xcur = xnext;
        if (ckpt != nullptr && live) {  // h at the half's last step: the checkpoint of the next half (NEXT-3)
          const int hsteps = C::KS;
          if (ch.vert) {
            const int t0 = j * C::K + half * C::KS;
            if (ln.own_v)
              *reinterpret_cast<float2*>(ckpt + ch.chain * ckstride + static_cast<int64_t>(t0 / hsteps) * ch.P +
                                         (ln.A + 2 * lane)) = make_float2(h[0], h[1]);
          } else {
            const int c0 = tile_start(ch, j, C::K) + cm * C::KS;
            const int t0 = ch.rev ? ch.L - c0 - C::KS : c0;
#pragma unroll
            for (int q = 0; q < kE; ++q) {
              const int r = ln.A + 32 * q + lane;
              if (ln.own_h[q] && r < ch.P)
                ckpt[ch.chain * ckstride + static_cast<int64_t>(t0 / hsteps) * ch.P + r] = h[q];
            }
          }
        }
        edge_publish(m.edge + par * kEdgeW * kXRow, warp, lane, ch.vert, h);
        if constexpr (kCl) {
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            if (!xgo(side, warp, pl.nwc, rank, pl.cl)) continue;
            const uint32_t tr = static_cast<uint32_t>(side == 0 ? rank - 1 : rank + 1);
            xput<T>(m, par, side, tr, 0, lane, ch.vert, h);
            xarrive(m, par, side, tr);
          }
        }
        named_bar(kBarEdge, nthreads);  // edges published; every warp has read this half's input rows
        edge_reload(m.edge + par * kEdgeW * kXRow, xs, ch.vert, h);
        if constexpr (kCl) {
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            if (!xgo(side, warp, pl.nwc, rank, pl.cl)) continue;
            xwait<T>(m, par, side, (xphase >> par) & 1u, 1);
            xget<T>(m, par, side, 0, lane, ch.vert, h);
          }
          xphase ^= 1u << par;
        }
        par ^= 1;
        if (!ch.vert && live) {  // new states in place over the x (kXG: lam) chunk of this half
#pragma unroll
          for (int q = 0; q < kE; ++q)
            if (ln.own_h[q])
              *reinterpret_cast<uint4*>(st + kOutSlot * kTile + (ln.hoff[q] ^ (static_cast<uint32_t>(cm) << 4))) = OUT[q];
        }
      }
      fence_proxy_async();  // in-place outputs -> visible to the storer's TMA (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&m.done[stage]));
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
    }
  }
  cluster_exit<kCl>();
}

template <typename T, int kPre, bool kCl, bool kLocal, bool kXG = false>
__global__ void __launch_bounds__((kMaxNWC + 2) * 32, 1) fwd_stream_kernel(const __grid_constant__ StreamArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Smem m = carve(smem_raw, A.plan);
  init_barriers<kCl>(m, A.plan);
  fwd_stream_body<T, kPre, kCl, kLocal, kXG>(A, m);
}

// ------------------------------------------------------------------------------ backward recurrence

// State carried between steps (reverse order): ea = a g, eb = b g, ec = c g of step t+1 at the lane's
// positions. g_t = dh_t + (b g)[r] + (a g)[r+1] + (c g)[r-1].
struct BwdState {
  float ea[kE], eb[kE], ec[kE];
};

template <int kPre>
__device__ __forceinline__ float bwd_math(float dh, float l, float m, float r, float nr, float nl, float& ea,
                                          float& eb, float& ec) {
  const float ge = (dh + eb) + (nr + nl);
  const float ig = kPre == kNormPre ? ge : norm_inv<kPre>((l + r) + m) * ge;
  ea = l * ig;
  eb = m * ig;
  ec = r * ig;
  return ge;
}

template <typename T, int kPre, bool kLocal>
__device__ __forceinline__ void bwd_half_vert(const Lanes<T>& ln, const uint8_t* p0, int stepb, T* gp,
                                              int64_t gstep, int t0, int L, BwdState& S, uint64_t pol, uint32_t rm) {
  constexpr int KS = Cfg<T>::KS;
  // steps t0 + KS - 1 down to t0; p0 / gp address step t0 + KS - 1
#pragma unroll
  for (int i = 0; i < KS; ++i) {
    const uint8_t* q = p0 + i * stepb;
    float dh[2], l[2], m[2], r[2];
    vload<T>(q + B_DH * kTile, dh);
    vload_tap<T>(q + B_WL * kTile, ln.s[0], l);
    vload_tap<T>(q + B_WM * kTile, ln.s[1], m);
    vload_tap<T>(q + B_WR * kTile, ln.s[2], r);
    const float nr1 = __shfl_down_sync(0xffffffffu, S.ea[0], 1);  // (a g) of the position above
    const float nl0 = __shfl_up_sync(0xffffffffu, S.ec[1], 1);    // (c g) of the position below
    const float ea0 = S.ea[1], ec1 = S.ec[0];
    float g[2];
    g[0] = bwd_math<kPre>(dh[0], l[0], m[0], r[0], ea0, nl0, S.ea[0], S.eb[0], S.ec[0]);
    g[1] = bwd_math<kPre>(dh[1], l[1], m[1], r[1], nr1, ec1, S.ea[1], S.eb[1], S.ec[1]);
    GStore<T, 2>::st_if(ln.own_v && t0 + KS - 1 - i < L, gp, g, pol);
    gp += gstep;
    if constexpr (kLocal) {  // segment start: g_{t-1} receives nothing from step t
      if ((rm >> i) & 1u) S.ea[0] = S.ea[1] = S.eb[0] = S.eb[1] = S.ec[0] = S.ec[1] = 0.f;
    }
  }
}

template <typename T, int kPre, bool kRev, bool kLocal, bool kMerged = false>
__device__ __forceinline__ void bwd_half_horiz(const Lanes<T>& ln, const uint8_t* st, int cm, int lane, BwdState& S,
                                               uint4 (&OG)[kE], uint32_t rm, float ms = 1.f) {
  constexpr int KS = Cfg<T>::KS;
  uint4 DH[kE], WL[kE], WM[kE], WR[kE], DY[kE];
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    const uint32_t off = ln.hoff[q] ^ (static_cast<uint32_t>(cm) << 4);
    DH[q] = *reinterpret_cast<const uint4*>(st + B_DH * kTile + off);
    WL[q] = *reinterpret_cast<const uint4*>(st + B_WL * kTile + off);
    WM[q] = *reinterpret_cast<const uint4*>(st + B_WM * kTile + off);
    WR[q] = *reinterpret_cast<const uint4*>(st + B_WR * kTile + off);
    if constexpr (kMerged) DY[q] = *reinterpret_cast<const uint4*>(st + B_DY * kTile + off);
  }
  float G_[kE][KS];
#pragma unroll
  for (int ss = KS - 1; ss >= 0; --ss) {  // scan order descending
    const int i = kRev ? KS - 1 - ss : ss;
    float nr[kE], nl[kE];
    slot_hi(S.ea, lane, nr);
    slot_lo(S.ec, lane, nl);
#pragma unroll
    for (int q = 0; q < kE; ++q)
      G_[q][i] = bwd_math<kPre>(kMerged ? ms * hget<T>(DH[q], i) * hget<T>(DY[q], i) : hget<T>(DH[q], i),
                                hget_tap<T>(WL[q], i, ln.s[0][q]),
                                hget_tap<T>(WM[q], i, ln.s[1][q]), hget_tap<T>(WR[q], i, ln.s[2][q]), nr[q], nl[q],
                                S.ea[q], S.eb[q], S.ec[q]);
    if constexpr (kLocal) {
      if ((rm >> (KS - 1 - ss)) & 1u) S.ea[0] = S.ea[1] = S.eb[0] = S.eb[1] = S.ec[0] = S.ec[1] = 0.f;
    }
  }
#pragma unroll
  for (int q = 0; q < kE; ++q) OG[q] = Pk<T>::pack(G_[q]);
}

template <typename T, int kPre, bool kCl, bool kLocal>
__global__ void __launch_bounds__((kMaxNWC + 2) * 32, 1) bwd_stream_kernel(const __grid_constant__ StreamArgs A) {
  // 32-bit work-item decode (experiments: GSPN built with -DGSPN_BS64 keeps the 64-bit one)
#ifdef GSPN_BS64
  constexpr bool kBS32 = false;
#else
  constexpr bool kBS32 = true;
#endif
  using C = Cfg<T>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Plan& pl = A.plan;
  const Smem m = carve(smem_raw, pl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  init_barriers<kCl>(m, pl);
  if (warp == pl.nwc) {
    if (lane == 0) {
      for (int o = 0; o < 2; ++o)
        for (int t = 0; t < B_NIN; ++t) asm volatile("prefetch.tensormap [%0];" ::"l"(&A.in[o][t]) : "memory");
      producer_loop<true, kCl, false, false, kBS32>(A, m.ring, m.full, m.empty);
    }
    cluster_exit<kCl>();
    return;
  }
  if (warp == pl.nwc + 1) {  // storer warp: horizontal tiles' g (written over the dh slot)
    if (lane == 0) {
      const int slots[1] = {B_DH};
      storer_loop<kCl, kBS32>(A, m.ring, m.done, m.empty, 1, slots, true);
    }
    cluster_exit<kCl>();
    return;
  }
  const uint64_t pol_vout = policy_of(pl.pol[3]);
  const int nthreads = pl.nwc * 32;
  const int64_t W = A.p.W;
  const int kchunk = static_cast<int>(A.p.kchunk);
  const int rank = kCl ? static_cast<int>(cluster_ctarank()) : 0;
  const XSrc xs = make_xsrc<T>(warp, pl.nwc, lane);
  uint32_t xphase = 0;
  int stage = 0, par = 0;
  uint32_t phase = 0;
  for (int64_t w = work_first<kCl>(pl); w < pl.nchains; w += work_stride<kCl>(pl)) {
    const Chain ch = make_chain<kCl, kBS32>(A.p, pl, w);
    const Lanes<T> ln = make_lanes<T, kCl>(pl, A.p, ch, warp, lane);
    T* gout = static_cast<T*>(A.g) + ln.vout;
    BwdState S;
#pragma unroll
    for (int e = 0; e < kE; ++e) S.ea[e] = S.eb[e] = S.ec[e] = 0.f;
    for (int jj = 0; jj < ch.j1 - ch.j0; ++jj) {
      const int j = ch.j1 - 1 - jj;
      mbar_wait_sleep(smem_u32(&m.full[stage]), phase);
      __syncwarp();  // reconverge after the per-thread spin: the shuffles below need no collective fallback
      uint8_t* st = m.ring + static_cast<size_t>(stage) * pl.stage_bytes;
#pragma unroll 1
      for (int half = 1; half >= 0; --half) {
        uint4 OG[kE];
        const int cm = ch.rev ? 1 - half : half;
        const bool live = !pl.null_compute && !half_outside_k<C::K>(ch, j, half, cm);
        if (live) {
          uint32_t rm = 0;
          if (ch.vert) {
            const int t0 = j * C::K + half * C::KS;          // first (lowest) step of the half
            const int tl = t0 + C::KS - 1;                     // processed first
            const int kkl = ch.rev ? C::K - 1 - (half * C::KS + C::KS - 1) : half * C::KS + C::KS - 1;
            const int rowl = ch.rev ? ch.L - 1 - tl : tl;
            const int vs = static_cast<int>(pl.vstep);
            if constexpr (kLocal) rm = reset_bits(rowl, ch.rev ? 1 : -1, !ch.rev, kchunk, C::KS);
            bwd_half_vert<T, kPre, kLocal>(ln, st + ln.voff + kkl * vs, ch.rev ? vs : -vs,
                                           gout + static_cast<int64_t>(rowl) * W, ch.rev ? W : -W, t0, ch.L, S,
                                           pol_vout, rm);
          } else {
            if constexpr (kLocal)
              rm = reset_bits(tile_start(ch, j, C::K) + cm * C::KS + (ch.rev ? 0 : C::KS - 1), ch.rev ? 1 : -1,
                              !ch.rev, kchunk, C::KS);
            if (ch.rev) bwd_half_horiz<T, kPre, true, kLocal>(ln, st, cm, lane, S, OG, rm);
            else bwd_half_horiz<T, kPre, false, kLocal>(ln, st, cm, lane, S, OG, rm);
          }
        }
        edge_publish(m.edge + 0 * kXArr + par * kEdgeW * kXRow, warp, lane, ch.vert, S.ea);
        edge_publish(m.edge + 1 * kXArr + par * kEdgeW * kXRow, warp, lane, ch.vert, S.eb);
        edge_publish(m.edge + 2 * kXArr + par * kEdgeW * kXRow, warp, lane, ch.vert, S.ec);
        if constexpr (kCl) {
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            if (!xgo(side, warp, pl.nwc, rank, pl.cl)) continue;
            const uint32_t tr = static_cast<uint32_t>(side == 0 ? rank - 1 : rank + 1);
            xput<T>(m, par, side, tr, 0, lane, ch.vert, S.ea);
            xput<T>(m, par, side, tr, 1, lane, ch.vert, S.eb);
            xput<T>(m, par, side, tr, 2, lane, ch.vert, S.ec);
            xarrive(m, par, side, tr);
          }
        }
        named_bar(kBarEdge, nthreads);  // edges published; every warp has read this half's input rows
        edge_reload(m.edge + 0 * kXArr + par * kEdgeW * kXRow, xs, ch.vert, S.ea);
        edge_reload(m.edge + 1 * kXArr + par * kEdgeW * kXRow, xs, ch.vert, S.eb);
        edge_reload(m.edge + 2 * kXArr + par * kEdgeW * kXRow, xs, ch.vert, S.ec);
        if constexpr (kCl) {
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            if (!xgo(side, warp, pl.nwc, rank, pl.cl)) continue;
            xwait<T>(m, par, side, (xphase >> par) & 1u, 3);
            xget<T>(m, par, side, 0, lane, ch.vert, S.ea);
            xget<T>(m, par, side, 1, lane, ch.vert, S.eb);
            xget<T>(m, par, side, 2, lane, ch.vert, S.ec);
          }
          xphase ^= 1u << par;
        }
        par ^= 1;
        if (!ch.vert && live) {
#pragma unroll
          for (int q = 0; q < kE; ++q)
            if (ln.own_h[q])
              *reinterpret_cast<uint4*>(st + B_DH * kTile + (ln.hoff[q] ^ (static_cast<uint32_t>(cm) << 4))) = OG[q];
        }
      }
      fence_proxy_async();  // in-place outputs -> visible to the storer's TMA (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&m.done[stage]));
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
    }
  }
  cluster_exit<kCl>();
}


// ------------------------------------------------------------------------------ fused backward (G = C)
//
// The adjoint recurrence above plus the tap gradients of a7 in the same pass: with g_t, the step's raw
// taps (l, m, r) and 1/S already in registers, and h_{t-1}[r-1..r+1] streamed in as one more tile,
//   u = g / S^2;  d1 = h[r-1] - h[r], d2 = h[r-1] - h[r+1], d3 = h[r] - h[r+1]   (h = h_{t-1})
//   dw_l = u (m d1 + r d2),  dw_m = u (r d3 - l d1),  dw_r = -u (l d2 + m d3)
// which is the Jacobian of SURVEY.md §8(a) a7 ((m + r) Da - m Db - r Dc) / S^2 etc. with Da = g h[r-1],
// Db = g h[r], Dc = g h[r+1], regrouped (pre-normalised taps: dw = (Da, Db, Dc)). Out-of-range taps get
// dw = 0. This removes the second read of w and the g round trip's w half that the split backward
// pays; dlam and dx (which sum over directions) follow in one elementwise pass (bwd_dx_kernel).

// Per-lane tap-range flags from the unpack selectors (an out-of-range tap unpacks to 0).
template <typename T>
__device__ __forceinline__ bool tap_on(const uint32_t (&m)[2]) {
  if constexpr (sizeof(T) == 2) return m[0] != kSelZero;
  else return m[0] != 0u;
}

template <int kPre>
__device__ __forceinline__ void dw_math(float g, float l, float m, float r, float hm1, float h0, float hp1, float& ol,
                                        float& om, float& orr) {
  if constexpr (kPre == kNormPre) {
    ol = g * hm1; om = g * h0; orr = g * hp1;
  } else {
    const float inv = norm_inv<kPre>((l + r) + m);
    const float u = g * inv * inv;
    const float d1 = hm1 - h0, d2 = hm1 - hp1, d3 = h0 - hp1;
    ol = u * fmaf(m, d1, r * d2);
    om = u * fmaf(r, d3, -l * d1);
    orr = -u * fmaf(l, d2, m * d3);
  }
}

template <typename T, int kPre, bool kLocal, bool kMerged = false>
__device__ __forceinline__ void bwd_half_vert_fused(const Lanes<T>& ln, const uint8_t* p0, int stepb, int64_t gofs,
                                                    int64_t gstep, int t0, int L, BwdState& S, uint64_t pol, T* gbase,
                                                    T* dwl, T* dwm, T* dwr, bool hl0, bool hr1, uint32_t rm,
                                                    float ms = 1.f) {
  constexpr int KS = Cfg<T>::KS;
#pragma unroll
  for (int i = 0; i < KS; ++i) {
    const uint8_t* q = p0 + i * stepb;
    float dh[2], l[2], m[2], r[2], hp[2];
    vload<T>(q + B_DH * kTile, dh);
    if constexpr (kMerged) {  // dh = s u dy (u in the dh slot)
      float dy[2];
      vload<T>(q + B_DY * kTile, dy);
      dh[0] *= ms * dy[0];
      dh[1] *= ms * dy[1];
    }
    vload_tap<T>(q + B_WL * kTile, ln.s[0], l);
    vload_tap<T>(q + B_WM * kTile, ln.s[1], m);
    vload_tap<T>(q + B_WR * kTile, ln.s[2], r);
    vload<T>(q + B_H0 * kTile, hp);  // h_{t-1} at the lane's two positions
    const float nr1 = __shfl_down_sync(0xffffffffu, S.ea[0], 1);
    const float nl0 = __shfl_up_sync(0xffffffffu, S.ec[1], 1);
    const float hleft = __shfl_up_sync(0xffffffffu, hp[1], 1);    // h_{t-1}[r0 - 1] (lane 0: a ghost)
    const float hright = __shfl_down_sync(0xffffffffu, hp[0], 1);  // h_{t-1}[r0 + 2] (lane 31: a ghost)
    const float ea0 = S.ea[1], ec1 = S.ec[0];
    float g[2], ol[2], om[2], orr[2];
    g[0] = bwd_math<kPre>(dh[0], l[0], m[0], r[0], ea0, nl0, S.ea[0], S.eb[0], S.ec[0]);
    g[1] = bwd_math<kPre>(dh[1], l[1], m[1], r[1], nr1, ec1, S.ea[1], S.eb[1], S.ec[1]);
    dw_math<kPre>(g[0], l[0], m[0], r[0], hleft, hp[0], hp[1], ol[0], om[0], orr[0]);
    dw_math<kPre>(g[1], l[1], m[1], r[1], hp[0], hp[1], hright, ol[1], om[1], orr[1]);
    ol[0] = hl0 ? ol[0] : 0.f;    // position r0 may be the chain's first (no left tap)
    orr[1] = hr1 ? orr[1] : 0.f;  // position r0 + 1 may be its last (no right tap)
    if constexpr (kLocal) {  // GSPN-local segment start: h_{t-1} was not propagated -> dw = 0, carry reset
      if ((rm >> i) & 1u) {
        ol[0] = ol[1] = om[0] = om[1] = orr[0] = orr[1] = 0.f;
        S.ea[0] = S.ea[1] = S.eb[0] = S.eb[1] = S.ec[0] = S.ec[1] = 0.f;
      }
    }
    const bool st = ln.own_v && t0 + KS - 1 - i < L;
    GStore<T, 2>::st_if(st, gbase + gofs, g, pol);
    GStore<T, 2>::st_if(st, dwl + gofs, ol, pol);
    GStore<T, 2>::st_if(st, dwm + gofs, om, pol);
    GStore<T, 2>::st_if(st, dwr + gofs, orr, pol);
    gofs += gstep;
  }
}

// Horizontal tap gradients of one half, after the edge barrier (every warp has read this half's input
// chunks, so each lane may overwrite its OWNED rows in place): g of the half (OG, already rounded to the
// I/O dtype like the split path's workspace g), the raw taps re-read from shared memory, and h_{t-1} =
// the chunk shifted by one column towards step t-1 -- elements of the same chunk plus one edge element of
// the spill chunk (the other chunk of this tile, or the neighbouring tile B_H1) -- for rows r-1, r, r+1.
template <typename T, int kPre, bool kRev>
__device__ __forceinline__ void dw_half_horiz(const Lanes<T>& ln, uint8_t* st, int cm, const uint4 (&OG)[kE],
                                              const uint32_t (&hrow)[kE][3], const bool (&hl)[kE],
                                              const bool (&hr)[kE]) {
  constexpr int KS = Cfg<T>::KS;
  // L2R (h_{t-1} = column c-1): cm 1 -> this tile's chunk 0; cm 0 -> tile B_H1 chunk 1.
  // R2L (column c+1):           cm 0 -> this tile's chunk 1; cm 1 -> tile B_H1 chunk 0.
  const bool own_tile = kRev ? cm == 0 : cm == 1;
  const uint32_t sp_slot = own_tile ? B_H0 * kTile : B_H1 * kTile;
  const uint32_t sp_chunk = static_cast<uint32_t>(cm ^ 1) << 4;
  const uint32_t cmx = static_cast<uint32_t>(cm) << 4;
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    if (!ln.own_h[q]) continue;
    const uint32_t off = ln.hoff[q] ^ cmx;
    const uint4 WL = *reinterpret_cast<const uint4*>(st + B_WL * kTile + off);
    const uint4 WM = *reinterpret_cast<const uint4*>(st + B_WM * kTile + off);
    const uint4 WR = *reinterpret_cast<const uint4*>(st + B_WR * kTile + off);
    uint4 Hc[3], Hs[3];  // rows r-1, r, r+1: this chunk of B_H0, and the spill chunk
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      Hc[a] = *reinterpret_cast<const uint4*>(st + B_H0 * kTile + (hrow[q][a] ^ cmx));
      Hs[a] = *reinterpret_cast<const uint4*>(st + sp_slot + (hrow[q][a] ^ sp_chunk));
    }
    float ol[KS], om[KS], orr[KS];
#pragma unroll
    for (int i = 0; i < KS; ++i) {
      float hv[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if constexpr (!kRev) hv[a] = i > 0 ? hget<T>(Hc[a], i - 1) : hget<T>(Hs[a], KS - 1);
        else hv[a] = i < KS - 1 ? hget<T>(Hc[a], i + 1) : hget<T>(Hs[a], 0);
      }
      dw_math<kPre>(hget<T>(OG[q], i), hget_tap<T>(WL, i, ln.s[0][q]), hget_tap<T>(WM, i, ln.s[1][q]),
                    hget_tap<T>(WR, i, ln.s[2][q]), hv[0], hv[1], hv[2], ol[i], om[i], orr[i]);
      ol[i] = hl[q] ? ol[i] : 0.f;
      orr[i] = hr[q] ? orr[i] : 0.f;
    }
    *reinterpret_cast<uint4*>(st + B_DH * kTile + off) = OG[q];
    *reinterpret_cast<uint4*>(st + B_WL * kTile + off) = Pk<T>::pack(ol);
    *reinterpret_cast<uint4*>(st + B_WM * kTile + off) = Pk<T>::pack(om);
    *reinterpret_cast<uint4*>(st + B_WR * kTile + off) = Pk<T>::pack(orr);
  }
}

// Pack helpers for the horizontal outputs built one element per step.
template <typename T> struct PkAcc;
template <> struct PkAcc<__nv_bfloat16> {
  uint32_t w[4];
  float pend;  // the first element of a pair, until its partner arrives (elements come pairwise, either order)
  // i compile-time after unrolling; `first`: i is the first of its pair to be produced
  __device__ __forceinline__ void put(int i, float v, bool first) {
    if (first) {
      pend = v;
    } else {
      const float lo = (i & 1) ? pend : v, hi = (i & 1) ? v : pend;
      w[i >> 1] = pack_bf16x2(lo, hi);  // one cvt.rn.bf16x2 per pair
    }
  }
  __device__ __forceinline__ uint4 get() const { return make_uint4(w[0], w[1], w[2], w[3]); }
};
template <> struct PkAcc<float> {
  uint32_t w[4];
  __device__ __forceinline__ void put(int i, float v, bool) { w[i] = __float_as_uint(v); }
  __device__ __forceinline__ uint4 get() const { return make_uint4(w[0], w[1], w[2], w[3]); }
};

// Horizontal half of the fused backward with the tap gradients in the recurrence (kHF): h_{t-1} of the
// lane's rows is the previous element of the lane's own h chunk; at the chunk edge it is the edge element
// of the neighbouring chunk towards step t-1 -- the h tile holds 48-byte rows, the tile's two chunks plus
// that neighbour (L2R: [chunk -1 | 0 | 1], R2L: [0 | 1 | +1]). The neighbouring rows' h_{t-1} come by
// shuffle; g and dw are packed per step and written in place after the half's barrier (the storer sends
// the 4 tiles).
template <typename T, int kPre, bool kRev, bool kMerged = false>
__device__ __forceinline__ void bwd_half_horiz_hf(const Lanes<T>& ln, const uint8_t* st, int cm, int lane, BwdState& S,
                                                  const bool (&hl)[kE], const bool (&hrr)[kE], uint4 (&OG)[kE],
                                                  uint4 (&OL)[kE], uint4 (&OM)[kE], uint4 (&OR)[kE], float ms = 1.f) {
  constexpr int KS = Cfg<T>::KS;
  uint4 DH[kE], WL[kE], WM[kE], WR[kE], HP[kE], DY[kE];
  float HE[kE];  // h_{t-1} of the half's first scan step (edge element of the neighbouring chunk)
  const uint32_t own = static_cast<uint32_t>(kRev ? cm : cm + 1) * 16u;
  const uint32_t edge = static_cast<uint32_t>(kRev ? cm + 1 : cm) * 16u + (kRev ? 0u : KS - 1u) * sizeof(T);
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    const uint32_t off = ln.hoff[q] ^ (static_cast<uint32_t>(cm) << 4);
    const uint32_t hrow = (ln.hoff[q] >> 5) * 48u;
    DH[q] = *reinterpret_cast<const uint4*>(st + B_DH * kTile + off);
    WL[q] = *reinterpret_cast<const uint4*>(st + B_WL * kTile + off);
    WM[q] = *reinterpret_cast<const uint4*>(st + B_WM * kTile + off);
    WR[q] = *reinterpret_cast<const uint4*>(st + B_WR * kTile + off);
    HP[q] = *reinterpret_cast<const uint4*>(st + B_H0 * kTile + hrow + own);
    HE[q] = to_f(*reinterpret_cast<const T*>(st + B_H0 * kTile + hrow + edge));
    if constexpr (kMerged) DY[q] = *reinterpret_cast<const uint4*>(st + B_DY * kTile + off);
  }
  PkAcc<T> ag[kE], al[kE], am[kE], ar[kE];
#pragma unroll
  for (int ss = KS - 1; ss >= 0; --ss) {  // scan order descending
    const int i = kRev ? KS - 1 - ss : ss;
    float nr[kE], nl[kE], hv[kE], hlo[kE], hhi[kE];
    slot_hi(S.ea, lane, nr);
    slot_lo(S.ec, lane, nl);
#pragma unroll
    for (int q = 0; q < kE; ++q)  // h_{t-1} at the lane's rows
      hv[q] = kRev ? (i < KS - 1 ? hget<T>(HP[q], i + 1) : HE[q]) : (i > 0 ? hget<T>(HP[q], i - 1) : HE[q]);
    slot_lo(hv, lane, hlo);
    slot_hi(hv, lane, hhi);
    const bool first = kRev ? (i & 1) == 0 : (i & 1) == 1;
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      const float l = hget_tap<T>(WL[q], i, ln.s[0][q]), m = hget_tap<T>(WM[q], i, ln.s[1][q]);
      const float r = hget_tap<T>(WR[q], i, ln.s[2][q]);
      const float dh = kMerged ? ms * hget<T>(DH[q], i) * hget<T>(DY[q], i) : hget<T>(DH[q], i);
      const float g = bwd_math<kPre>(dh, l, m, r, nr[q], nl[q], S.ea[q], S.eb[q], S.ec[q]);
      float ol, om, orr;
      dw_math<kPre>(g, l, m, r, hlo[q], hv[q], hhi[q], ol, om, orr);
      ag[q].put(i, g, first);
      al[q].put(i, hl[q] ? ol : 0.f, first);
      am[q].put(i, om, first);
      ar[q].put(i, hrr[q] ? orr : 0.f, first);
    }
  }
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    OG[q] = ag[q].get();
    OL[q] = al[q].get();
    OM[q] = am[q].get();
    OR[q] = ar[q].get();
  }
}

template <typename T, int kPre, bool kMerged = false, bool kHF = false>
__device__ void producer_fused(const StreamArgs& A, uint8_t* ring, uint64_t* full, uint64_t* empty) {
  const Plan& pl = A.plan;
  const uint64_t pol_vin = policy_of(pl.pol[1]);
  const uint64_t pol_hin = policy_of(pl.pol[2]);
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t w = blockIdx.x; w < pl.nchains; w += gridDim.x) {
    const Chain ch = make_chain<false>(A.p, pl, w);
    const int chain = static_cast<int>(ch.chain);
    for (int jj = 0; jj < ch.j1 - ch.j0; ++jj) {
      const int j = ch.j1 - 1 - jj;
      mbar_wait_sleep(smem_u32(&empty[stage]), phase ^ 1);
      const uint32_t fb = smem_u32(&full[stage]);
      mbar_arrive_tx(fb, ch.vert ? pl.tx_v : pl.tx_h);
      const int s0 = tile_start(ch, j, pl.K);
      const uint32_t st = smem_u32(ring + static_cast<size_t>(stage) * pl.stage_bytes);
      const uint64_t pol = ch.vert ? pol_vin : pol_hin;
      for (int t = 0; t < B_NIN; ++t) {
        const uint32_t dst = st + t * pl.tile_bytes;
        if (pl.npack > 1) {  // packed chains: one 3D box, vertical (W, planes, rows), horizontal (cols, H, planes)
          if (ch.vert) tma_load3(dst, &A.in[0][t], 0, chain, s0, fb, pol);
          else tma_load3(dst, &A.in[1][t], s0, 0, chain, fb, pol);
        } else if (ch.vert) {
          for (int q = 0; q < pl.nbw; ++q)
            tma_load3(dst + q * pl.K * pl.bw * pl.es, &A.in[0][t], q * pl.bw, s0, chain, fb, pol);
        } else {
          for (int q = 0; q < pl.nbh; ++q)
            tma_load3(dst + q * pl.bh * 32, &A.in[1][t], s0, q * pl.bh, chain, fb, pol);
        }
      }
      if (ch.vert) {  // h rows one step earlier: T2B row - 1, B2T row + 1 (out of range: zero = h_{-1})
        const int sh = ch.rev ? s0 + 1 : s0 - 1;
        const uint32_t dst = st + B_H0 * pl.tile_bytes;
        if (pl.npack > 1) {
          tma_load3(dst, &A.in[0][B_H0], 0, chain, sh, fb, pol);
        } else {
          for (int q = 0; q < pl.nbw; ++q)
            tma_load3(dst + q * pl.K * pl.bw * pl.es, &A.in[0][B_H0], q * pl.bw, sh, chain, fb, pol);
        }
      } else if (kHF) {  // h of the tile's columns plus the 16-byte chunk towards step t-1 (48-byte rows, no
                         // swizzle): TMA needs a 16-byte aligned inner coordinate, so the box cannot start one
                         // column earlier; L2R [s0 - KS, s0 + K), R2L [s0, s0 + K + KS) (edges: zero fill = h_{-1})
        const int sh = ch.rev ? s0 : s0 - pl.K / 2;
        if (pl.npack > 1) {
          tma_load3(st + B_H0 * pl.tile_bytes, &A.in[1][B_H0], sh, 0, chain, fb, pol);
        } else {
          for (int q = 0; q < pl.nbh; ++q)
            tma_load3(st + B_H0 * pl.tile_bytes + q * pl.bh * 48, &A.in[1][B_H0], sh, q * pl.bh, chain, fb, pol);
        }
      } else if (pl.fuse_h) {  // this tile's columns and the neighbouring tile towards step t-1 (zero fill)
        const int sn = ch.rev ? s0 + pl.K : s0 - pl.K;
        for (int q = 0; q < pl.nbh; ++q) {
          tma_load3(st + B_H0 * pl.tile_bytes + q * pl.bh * 32, &A.in[1][B_H0], s0, q * pl.bh, chain, fb, pol);
          tma_load3(st + B_H1 * pl.tile_bytes + q * pl.bh * 32, &A.in[1][B_H0], sn, q * pl.bh, chain, fb, pol);
        }
      }
      if constexpr (kMerged) {  // dy of the plane (shared by the directions: plane index b C + c)
        const int plane = static_cast<int>(ch.bc);
        const uint32_t dst = st + B_DY * pl.tile_bytes;
        const uint64_t pold = policy_of(pl.pol[0]);
        if (pl.npack > 1) {
          if (ch.vert) tma_load3(dst, &A.in[0][B_DY], 0, plane, s0, fb, pold);
          else tma_load3(dst, &A.in[1][B_DY], s0, 0, plane, fb, pold);
        } else if (ch.vert) {
          for (int q = 0; q < pl.nbw; ++q)
            tma_load3(dst + q * pl.K * pl.bw * pl.es, &A.in[0][B_DY], q * pl.bw, s0, plane, fb, pold);
        } else {
          for (int q = 0; q < pl.nbh; ++q)
            tma_load3(dst + q * pl.bh * 32, &A.in[1][B_DY], s0, q * pl.bh, plane, fb, pold);
        }
      }
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
    }
  }
}

// Body of the fused backward recurrence (every role returns from here when its work is done); the
// barriers of `m` must be initialised. Shared by bwd_fused_kernel and the single-launch bwd_one_kernel.
template <typename T, int kPre, bool kLocal, bool kMerged = false, bool kHF = false>
__device__ __forceinline__ void bwd_fused_body(const StreamArgs& A, const Smem& m) {
  using C = Cfg<T>;
  const Plan& pl = A.plan;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == pl.nwc) {
    if (lane == 0) {
      for (int o = 0; o < 2; ++o)
        for (int t = 0; t < B_H1; ++t) asm volatile("prefetch.tensormap [%0];" ::"l"(&A.in[o][t]) : "memory");
      producer_fused<T, kPre, kMerged, kHF>(A, m.ring, m.full, m.empty);
    }
    return;
  }
  if (warp == pl.nwc + 1) {  // storer: horizontal tiles' g and dw_l/m/r (written over dh, w_l, w_m, w_r)
    if (lane == 0) {
      const int slots[4] = {B_DH, B_WL, B_WM, B_WR};
      storer_loop<false>(A, m.ring, m.done, m.empty, (pl.fuse_h || kHF) ? 4 : 1, slots, true);
    }
    return;
  }
  const uint64_t pol_vout = policy_of(pl.pol[3]);
  const int nthreads = pl.nwc * 32;
  const int64_t W = A.p.W;
  const XSrc xs = make_xsrc<T>(warp, pl.nwc, lane);
  T* const gbase = static_cast<T*>(A.g);
  T* const dwl = static_cast<T*>(A.p.dwl);
  T* const dwm = static_cast<T*>(A.p.dwm);
  T* const dwr = static_cast<T*>(A.p.dwr);
  const int kchunk = static_cast<int>(A.p.kchunk);
  const float mscale = A.p.merge_scale;
  int stage = 0, par = 0;
  uint32_t phase = 0;
  for (int64_t w = blockIdx.x; w < pl.nchains; w += gridDim.x) {
    const Chain ch = make_chain<false>(A.p, pl, w);
    const Lanes<T> ln = make_lanes<T, false>(pl, A.p, ch, warp, lane);
    // tap-range flags and the swizzled offsets of rows r-1, r, r+1 (horizontal slots)
    const bool hl0 = tap_on<T>(ln.s[0][0]), hr1 = tap_on<T>(ln.s[2][1]);
    bool hl[kE], hr[kE];
    uint32_t hrow[kE][3];
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      hl[q] = tap_on<T>(ln.s[0][q]);
      hr[q] = tap_on<T>(ln.s[2][q]);
      const int rt = ln.A + 32 * q + lane;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        int rr = rt - 1 + a;
        rr = rr < 0 ? 0 : (rr >= kPpad ? kPpad - 1 : rr);
        const uint32_t rc = static_cast<uint32_t>(rr);
        hrow[q][a] = rc * 32 + (((rc >> 2) & 1u) << 4);
      }
    }
    BwdState S;
#pragma unroll
    for (int e = 0; e < kE; ++e) S.ea[e] = S.eb[e] = S.ec[e] = 0.f;
    for (int jj = 0; jj < ch.j1 - ch.j0; ++jj) {
      const int j = ch.j1 - 1 - jj;
      mbar_wait_sleep(smem_u32(&m.full[stage]), phase);
      __syncwarp();
      uint8_t* st = m.ring + static_cast<size_t>(stage) * pl.stage_bytes;
#pragma unroll 1
      for (int half = 1; half >= 0; --half) {
        uint4 OG[kE], OL[kE], OM[kE], OR[kE];
        const int cm = ch.rev ? 1 - half : half;
        const bool live = !pl.null_compute && !half_outside_k<C::K>(ch, j, half, cm);
        if (live) {
          uint32_t rm = 0;
          if (ch.vert) {
            const int t0 = j * C::K + half * C::KS;
            const int tl = t0 + C::KS - 1;
            const int kkl = ch.rev ? C::K - 1 - (half * C::KS + C::KS - 1) : half * C::KS + C::KS - 1;
            const int rowl = ch.rev ? ch.L - 1 - tl : tl;
            const int vs = static_cast<int>(pl.vstep);
            if constexpr (kLocal) rm = reset_bits(rowl, ch.rev ? 1 : -1, !ch.rev, kchunk, C::KS);
            bwd_half_vert_fused<T, kPre, kLocal, kMerged>(ln, st + ln.voff + kkl * vs, ch.rev ? vs : -vs,
                                                          ln.vout + static_cast<int64_t>(rowl) * W, ch.rev ? W : -W, t0,
                                                          ch.L, S, pol_vout, gbase, dwl, dwm, dwr, hl0, hr1, rm, mscale);
          } else {
            if constexpr (kLocal)
              rm = reset_bits(tile_start(ch, j, C::K) + cm * C::KS + (ch.rev ? 0 : C::KS - 1), ch.rev ? 1 : -1,
                              !ch.rev, kchunk, C::KS);
            if constexpr (kHF) {
              if (ch.rev) bwd_half_horiz_hf<T, kPre, true, kMerged>(ln, st, cm, lane, S, hl, hr, OG, OL, OM, OR, mscale);
              else bwd_half_horiz_hf<T, kPre, false, kMerged>(ln, st, cm, lane, S, hl, hr, OG, OL, OM, OR, mscale);
            } else {
              if (ch.rev) bwd_half_horiz<T, kPre, true, kLocal, kMerged>(ln, st, cm, lane, S, OG, rm, mscale);
              else bwd_half_horiz<T, kPre, false, kLocal, kMerged>(ln, st, cm, lane, S, OG, rm, mscale);
            }
          }
        }
        edge_publish(m.edge + 0 * kXArr + par * kEdgeW * kXRow, warp, lane, ch.vert, S.ea);
        edge_publish(m.edge + 1 * kXArr + par * kEdgeW * kXRow, warp, lane, ch.vert, S.eb);
        edge_publish(m.edge + 2 * kXArr + par * kEdgeW * kXRow, warp, lane, ch.vert, S.ec);
        named_bar(kBarEdge, nthreads);  // edges published; every warp has read this half's input rows
        edge_reload(m.edge + 0 * kXArr + par * kEdgeW * kXRow, xs, ch.vert, S.ea);
        edge_reload(m.edge + 1 * kXArr + par * kEdgeW * kXRow, xs, ch.vert, S.eb);
        edge_reload(m.edge + 2 * kXArr + par * kEdgeW * kXRow, xs, ch.vert, S.ec);
        par ^= 1;
        if (!ch.vert && live && kHF) {  // g and dw in place over dh / w chunks (storer: 4 tiles)
#pragma unroll
          for (int q = 0; q < kE; ++q) {
            if (!ln.own_h[q]) continue;
            const uint32_t off = ln.hoff[q] ^ (static_cast<uint32_t>(cm) << 4);
            *reinterpret_cast<uint4*>(st + B_DH * kTile + off) = OG[q];
            *reinterpret_cast<uint4*>(st + B_WL * kTile + off) = OL[q];
            *reinterpret_cast<uint4*>(st + B_WM * kTile + off) = OM[q];
            *reinterpret_cast<uint4*>(st + B_WR * kTile + off) = OR[q];
          }
        } else if (!ch.vert && live) {
          if (pl.fuse_h) {  // tap gradients; g and dw in place over this half's dh / w chunks
            if (ch.rev) dw_half_horiz<T, kPre, true>(ln, st, cm, OG, hrow, hl, hr);
            else dw_half_horiz<T, kPre, false>(ln, st, cm, OG, hrow, hl, hr);
          } else {  // g only (the output kernel forms these chains' dw): in place over the dh chunk
#pragma unroll
            for (int q = 0; q < kE; ++q)
              if (ln.own_h[q])
                *reinterpret_cast<uint4*>(st + B_DH * kTile + (ln.hoff[q] ^ (static_cast<uint32_t>(cm) << 4))) = OG[q];
          }
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&m.done[stage]));
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
    }
  }
}

// ------------------------------------------------------------------------------ recompute-h backward
//
// NEXT-3: the backward reads fp32 checkpoints of h (one per half-tile,
// written by the forward, gspn_fwd_ckpt) instead of the stored h. Per half-tile, in the reverse sweep,
// every lane first re-runs the forward recurrence (Eq. 1) over the half's first KS-1 steps from the
// checkpoint h_{t0-1} -- x, lam and the taps come with the stage -- keeping h_{t0-1} .. h_{t0+KS-2} in
// registers, then runs the adjoint steps with the tap gradients of BOTH orientations in the recurrence
// (dw = u (m d1 + r d2) etc. from h_{t-1} of the lane and its neighbours by shuffle). A warp's window
// (64 positions, 48 owned) starts from exact checkpoint values everywhere, so after KS - 1 <= 7 recomputed
// steps its owned positions and their neighbours are still exact (GH = KS). The output phase then forms
// only dlam and dx for every direction. Unpacked, unsplit chains with H, W multiples of K.
enum BwdRcIn { R_DH = 0, R_WL, R_WM, R_WR, R_X, R_LAM, R_NIN };

template <typename T, int kPre>
__device__ void producer_rc(const StreamArgs& A, uint8_t* ring, uint64_t* full, uint64_t* empty) {
  const Plan& pl = A.plan;
  const uint64_t pol_vin = policy_of(pl.pol[1]);
  const uint64_t pol_hin = policy_of(pl.pol[2]);
  const uint64_t pol_x = policy_of(pl.pol[0]);
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t w = blockIdx.x; w < pl.nchains; w += gridDim.x) {
    const Chain ch = make_chain<false>(A.p, pl, w);
    for (int jj = 0; jj < ch.j1 - ch.j0; ++jj) {
      const int j = ch.j1 - 1 - jj;
      mbar_wait_sleep(smem_u32(&empty[stage]), phase ^ 1);
      const uint32_t fb = smem_u32(&full[stage]);
      mbar_arrive_tx(fb, ch.vert ? pl.tx_v : pl.tx_h);
      const int s0 = tile_start(ch, j, pl.K);
      const uint32_t st = smem_u32(ring + static_cast<size_t>(stage) * pl.stage_bytes);
      for (int t = 0; t < R_NIN; ++t) {
        const int plane = static_cast<int>(t == R_X ? ch.bc : ch.chain);
        const uint64_t pol = t == R_X ? pol_x : (ch.vert ? pol_vin : pol_hin);
        const uint32_t dst = st + t * pl.tile_bytes;
        if (ch.vert) {
          for (int q = 0; q < pl.nbw; ++q) tma_load3(dst + q * pl.K * pl.bw * pl.es, &A.in[0][t], q * pl.bw, s0, plane, fb, pol);
        } else {
          for (int q = 0; q < pl.nbh; ++q) tma_load3(dst + q * pl.bh * 32, &A.in[1][t], s0, q * pl.bh, plane, fb, pol);
        }
      }
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
    }
  }
}

// Vertical half: pf = the lane's operands at the half's FIRST scan step, sf = +-row stride in scan order.
template <typename T, int kPre>
__device__ __forceinline__ void rc_half_vert(const Lanes<T>& ln, const uint8_t* pf, int sf, int64_t gofs_last,
                                             int64_t gstep, BwdState& S, uint64_t pol, T* gbase, T* dwl, T* dwm,
                                             T* dwr, bool hl0, bool hr1, const float (&hck)[2]) {
  constexpr int KS = Cfg<T>::KS;
  float hr[KS][2];  // hr[s] = h_{t0-1+s}
  hr[0][0] = hck[0];
  hr[0][1] = hck[1];
#pragma unroll
  for (int s = 0; s < KS - 1; ++s) {
    const uint8_t* q = pf + s * sf;
    float x[2], lam[2], l[2], m[2], r[2];
    vload<T>(q + R_X * kTile, x);
    vload<T>(q + R_LAM * kTile, lam);
    vload_tap<T>(q + R_WL * kTile, ln.s[0], l);
    vload_tap<T>(q + R_WM * kTile, ln.s[1], m);
    vload_tap<T>(q + R_WR * kTile, ln.s[2], r);
    const float left = __shfl_up_sync(0xffffffffu, hr[s][1], 1);
    const float right = __shfl_down_sync(0xffffffffu, hr[s][0], 1);
    hr[s + 1][0] = fwd_math<kPre>(x[0], lam[0], l[0], m[0], r[0], left, hr[s][0], hr[s][1]);
    hr[s + 1][1] = fwd_math<kPre>(x[1], lam[1], l[1], m[1], r[1], hr[s][0], hr[s][1], right);
  }
  int64_t gofs = gofs_last;
#pragma unroll
  for (int i = 0; i < KS; ++i) {  // adjoint, steps t0 + KS - 1 down to t0
    const int s = KS - 1 - i;
    const uint8_t* q = pf + s * sf;
    float dh[2], l[2], m[2], r[2];
    vload<T>(q + R_DH * kTile, dh);
    vload_tap<T>(q + R_WL * kTile, ln.s[0], l);
    vload_tap<T>(q + R_WM * kTile, ln.s[1], m);
    vload_tap<T>(q + R_WR * kTile, ln.s[2], r);
    const float nr1 = __shfl_down_sync(0xffffffffu, S.ea[0], 1);
    const float nl0 = __shfl_up_sync(0xffffffffu, S.ec[1], 1);
    const float hleft = __shfl_up_sync(0xffffffffu, hr[s][1], 1);    // h_{t-1}[r0 - 1]
    const float hright = __shfl_down_sync(0xffffffffu, hr[s][0], 1);  // h_{t-1}[r0 + 2]
    const float ea0 = S.ea[1], ec1 = S.ec[0];
    float g[2], ol[2], om[2], orr[2];
    g[0] = bwd_math<kPre>(dh[0], l[0], m[0], r[0], ea0, nl0, S.ea[0], S.eb[0], S.ec[0]);
    g[1] = bwd_math<kPre>(dh[1], l[1], m[1], r[1], nr1, ec1, S.ea[1], S.eb[1], S.ec[1]);
    dw_math<kPre>(g[0], l[0], m[0], r[0], hleft, hr[s][0], hr[s][1], ol[0], om[0], orr[0]);
    dw_math<kPre>(g[1], l[1], m[1], r[1], hr[s][0], hr[s][1], hright, ol[1], om[1], orr[1]);
    ol[0] = hl0 ? ol[0] : 0.f;
    orr[1] = hr1 ? orr[1] : 0.f;
    GStore<T, 2>::st_if(ln.own_v, gbase + gofs, g, pol);
    GStore<T, 2>::st_if(ln.own_v, dwl + gofs, ol, pol);
    GStore<T, 2>::st_if(ln.own_v, dwm + gofs, om, pol);
    GStore<T, 2>::st_if(ln.own_v, dwr + gofs, orr, pol);
    gofs += gstep;
  }
}

template <typename T, int kPre, bool kRev>
__device__ __forceinline__ void rc_half_horiz(const Lanes<T>& ln, const uint8_t* st, int cm, int lane, BwdState& S,
                                              const float (&hck)[kE], const bool (&hl)[kE], const bool (&hrr)[kE],
                                              uint4 (&OG)[kE], uint4 (&OL)[kE], uint4 (&OM)[kE], uint4 (&OR)[kE]) {
  constexpr int KS = Cfg<T>::KS;
  uint4 DH[kE], WL[kE], WM[kE], WR[kE], X[kE], LAM[kE];
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    const uint32_t off = ln.hoff[q] ^ (static_cast<uint32_t>(cm) << 4);
    DH[q] = *reinterpret_cast<const uint4*>(st + R_DH * kTile + off);
    WL[q] = *reinterpret_cast<const uint4*>(st + R_WL * kTile + off);
    WM[q] = *reinterpret_cast<const uint4*>(st + R_WM * kTile + off);
    WR[q] = *reinterpret_cast<const uint4*>(st + R_WR * kTile + off);
    X[q] = *reinterpret_cast<const uint4*>(st + R_X * kTile + off);
    LAM[q] = *reinterpret_cast<const uint4*>(st + R_LAM * kTile + off);
  }
  float hr[KS][kE];  // hr[s] = h_{t0-1+s} (scan order)
#pragma unroll
  for (int q = 0; q < kE; ++q) hr[0][q] = hck[q];
#pragma unroll
  for (int s = 0; s < KS - 1; ++s) {
    const int i = kRev ? KS - 1 - s : s;
    float lo[kE], hi[kE];
    slot_lo(hr[s], lane, lo);
    slot_hi(hr[s], lane, hi);
#pragma unroll
    for (int q = 0; q < kE; ++q)
      hr[s + 1][q] = fwd_math<kPre>(hget<T>(X[q], i), hget<T>(LAM[q], i), hget_tap<T>(WL[q], i, ln.s[0][q]),
                                    hget_tap<T>(WM[q], i, ln.s[1][q]), hget_tap<T>(WR[q], i, ln.s[2][q]), lo[q],
                                    hr[s][q], hi[q]);
  }
  PkAcc<T> ag[kE], al[kE], am[kE], ar[kE];
#pragma unroll
  for (int ss = KS - 1; ss >= 0; --ss) {  // adjoint, scan order descending
    const int i = kRev ? KS - 1 - ss : ss;
    float nr[kE], nl[kE], hlo[kE], hhi[kE];
    slot_hi(S.ea, lane, nr);
    slot_lo(S.ec, lane, nl);
    slot_lo(hr[ss], lane, hlo);  // h_{t-1}[r-1]
    slot_hi(hr[ss], lane, hhi);  // h_{t-1}[r+1]
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      const float l = hget_tap<T>(WL[q], i, ln.s[0][q]), m = hget_tap<T>(WM[q], i, ln.s[1][q]);
      const float r = hget_tap<T>(WR[q], i, ln.s[2][q]);
      const float g = bwd_math<kPre>(hget<T>(DH[q], i), l, m, r, nr[q], nl[q], S.ea[q], S.eb[q], S.ec[q]);
      float ol, om, orr;
      dw_math<kPre>(g, l, m, r, hlo[q], hr[ss][q], hhi[q], ol, om, orr);
      const bool first = kRev ? (i & 1) == 0 : (i & 1) == 1;  // ss descends: i descends (L2R) / ascends (R2L)
      ag[q].put(i, g, first);
      al[q].put(i, hl[q] ? ol : 0.f, first);
      am[q].put(i, om, first);
      ar[q].put(i, hrr[q] ? orr : 0.f, first);
    }
  }
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    OG[q] = ag[q].get();
    OL[q] = al[q].get();
    OM[q] = am[q].get();
    OR[q] = ar[q].get();
  }
}

template <typename T, int kPre>
__device__ __forceinline__ void bwd_rc_body(const StreamArgs& A, const Smem& m) {
  using C = Cfg<T>;
  const Plan& pl = A.plan;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == pl.nwc) {
    if (lane == 0) {
      for (int o = 0; o < 2; ++o)
        for (int t = 0; t < R_NIN; ++t) asm volatile("prefetch.tensormap [%0];" ::"l"(&A.in[o][t]) : "memory");
      producer_rc<T, kPre>(A, m.ring, m.full, m.empty);
    }
    return;
  }
  if (warp == pl.nwc + 1) {  // storer: horizontal tiles' g and dw (in place over dh and the taps)
    if (lane == 0) {
      const int slots[4] = {R_DH, R_WL, R_WM, R_WR};
      storer_loop<false>(A, m.ring, m.done, m.empty, 4, slots, true);
    }
    return;
  }
  const uint64_t pol_vout = policy_of(pl.pol[3]);
  const int nthreads = pl.nwc * 32;
  const int64_t W = A.p.W;
  const XSrc xs = make_xsrc<T>(warp, pl.nwc, lane);
  T* const gbase = static_cast<T*>(A.g);
  T* const dwl = static_cast<T*>(A.p.dwl);
  T* const dwm = static_cast<T*>(A.p.dwm);
  T* const dwr = static_cast<T*>(A.p.dwr);
  const float* const ckpt = A.p.ckpt;
  const int64_t ckstride = A.p.H * A.p.W / C::KS;
  int stage = 0, par = 0;
  uint32_t phase = 0;
  for (int64_t w = blockIdx.x; w < pl.nchains; w += gridDim.x) {
    const Chain ch = make_chain<false>(A.p, pl, w);
    const Lanes<T> ln = make_lanes<T, false>(pl, A.p, ch, warp, lane);
    const bool hl0 = tap_on<T>(ln.s[0][0]), hr1 = tap_on<T>(ln.s[2][1]);
    bool hl[kE], hrr[kE];
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      hl[q] = tap_on<T>(ln.s[0][q]);
      hrr[q] = tap_on<T>(ln.s[2][q]);
    }
    const float* ckc = ckpt + ch.chain * ckstride;
    const int r0 = ln.A + 2 * lane;                 // vertical: the lane's first position
    const bool v_in = r0 >= 0 && r0 < ch.P;
    // checkpoint h_{t0-1} of the half with first scan step t0 (0 at t0 = 0): loaded one half ahead
    auto ck_load = [&](int t0, float (&o)[2]) {
      o[0] = o[1] = 0.f;
      if (t0 <= 0) return;
      const float* row = ckc + static_cast<int64_t>(t0 / C::KS - 1) * ch.P;
      if (ch.vert) {
        if (v_in) {
          const float2 u = __ldcg(reinterpret_cast<const float2*>(row + r0));
          o[0] = u.x;
          o[1] = u.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < kE; ++q) {
          const int r = ln.A + 32 * q + lane;
          if (r >= 0 && r < ch.P) o[q] = __ldcg(row + r);
        }
      }
    };
    auto first_step = [&](int j, int half) {  // scan index of the half's first step
      if (ch.vert) return j * C::K + half * C::KS;
      const int cm = ch.rev ? 1 - half : half;
      const int c0 = tile_start(ch, j, C::K) + cm * C::KS;
      return ch.rev ? ch.L - c0 - C::KS : c0;
    };
    float ckn[2];
    ck_load(first_step(ch.ntiles - 1, 1), ckn);
    BwdState S;
#pragma unroll
    for (int e = 0; e < kE; ++e) S.ea[e] = S.eb[e] = S.ec[e] = 0.f;
    for (int jj = 0; jj < ch.j1 - ch.j0; ++jj) {
      const int j = ch.j1 - 1 - jj;
      mbar_wait_sleep(smem_u32(&m.full[stage]), phase);
      __syncwarp();
      uint8_t* st = m.ring + static_cast<size_t>(stage) * pl.stage_bytes;
#pragma unroll 1
      for (int half = 1; half >= 0; --half) {
        const int cm = ch.rev ? 1 - half : half;
        const float ckc_[2] = {ckn[0], ckn[1]};
        {  // the next half's checkpoint (reverse order), in flight while this half computes
          const int jn = half == 1 ? j : j - 1, hn = half ^ 1;
          if (jn >= 0) ck_load(first_step(jn, hn), ckn);
        }
        uint4 OG[kE], OL[kE], OM[kE], OR[kE];
        const bool live = !pl.null_compute;
        if (live) {
          if (ch.vert) {
            const int t0 = j * C::K + half * C::KS;
            const int kkf = ch.rev ? C::K - 1 - half * C::KS : half * C::KS;  // tile row of the first step
            const int vs = static_cast<int>(pl.vstep);
            const int tl = t0 + C::KS - 1;
            const int rowl = ch.rev ? ch.L - 1 - tl : tl;
            rc_half_vert<T, kPre>(ln, st + ln.voff + kkf * vs, ch.rev ? -vs : vs,
                                  ln.vout + static_cast<int64_t>(rowl) * W, ch.rev ? W : -W, S, pol_vout, gbase, dwl,
                                  dwm, dwr, hl0, hr1, ckc_);
          } else {
            if (ch.rev) rc_half_horiz<T, kPre, true>(ln, st, cm, lane, S, ckc_, hl, hrr, OG, OL, OM, OR);
            else rc_half_horiz<T, kPre, false>(ln, st, cm, lane, S, ckc_, hl, hrr, OG, OL, OM, OR);
          }
        }
        edge_publish(m.edge + 0 * kXArr + par * kEdgeW * kXRow, warp, lane, ch.vert, S.ea);
        edge_publish(m.edge + 1 * kXArr + par * kEdgeW * kXRow, warp, lane, ch.vert, S.eb);
        edge_publish(m.edge + 2 * kXArr + par * kEdgeW * kXRow, warp, lane, ch.vert, S.ec);
        named_bar(kBarEdge, nthreads);  // edges published; every warp has read this half's input rows
        edge_reload(m.edge + 0 * kXArr + par * kEdgeW * kXRow, xs, ch.vert, S.ea);
        edge_reload(m.edge + 1 * kXArr + par * kEdgeW * kXRow, xs, ch.vert, S.eb);
        edge_reload(m.edge + 2 * kXArr + par * kEdgeW * kXRow, xs, ch.vert, S.ec);
        par ^= 1;
        if (!ch.vert && live) {  // g and dw in place over this half's dh / tap chunks (owned rows)
#pragma unroll
          for (int q = 0; q < kE; ++q) {
            if (!ln.own_h[q]) continue;
            const uint32_t off = ln.hoff[q] ^ (static_cast<uint32_t>(cm) << 4);
            *reinterpret_cast<uint4*>(st + R_DH * kTile + off) = OG[q];
            *reinterpret_cast<uint4*>(st + R_WL * kTile + off) = OL[q];
            *reinterpret_cast<uint4*>(st + R_WM * kTile + off) = OM[q];
            *reinterpret_cast<uint4*>(st + R_WR * kTile + off) = OR[q];
          }
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&m.done[stage]));
      if (++stage == pl.nstages) { stage = 0; phase ^= 1; }
    }
  }
}

template <typename T, int kPre, bool kLocal>
__global__ void __launch_bounds__((kMaxNWC + 2) * 32, 1) bwd_fused_kernel(const __grid_constant__ StreamArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Smem m = carve(smem_raw, A.plan);
  init_barriers<false>(m, A.plan);
  bwd_fused_body<T, kPre, kLocal>(A, m);
}

// dlam_k = g_k x and dx = sum_k g_k lam_k (a7), elementwise over [B, C, H, W] with all D directions per
// thread; 16-byte vectors, streaming loads / stores (HBM-bound: s (1 + 4D) reads + s (D + 1) writes).
template <typename T, int D>
__global__ void __launch_bounds__(256) bwd_dx_kernel(const T* __restrict__ x, const T* __restrict__ lam,
                                                     const T* __restrict__ g, T* __restrict__ dlam,
                                                     T* __restrict__ dx, int64_t N, int64_t nv) {
  constexpr int V = 16 / sizeof(T);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 gq[D], lq[D];
    const uint4 xq = ld_nc_v4(x + i * V);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      gq[k] = ld_nc_v4(g + k * N + i * V);
      lq[k] = ld_nc_v4(lam + k * N + i * V);
    }
    float xv[V], acc[V];
#pragma unroll
    for (int e = 0; e < V; ++e) {
      xv[e] = hget<T>(xq, e);
      acc[e] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      float dl[V];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const float gv = hget<T>(gq[k], e);
        dl[e] = gv * xv[e];
        acc[e] = fmaf(gv, hget<T>(lq[k], e), acc[e]);
      }
      st_cs_v4(dlam + k * N + i * V, Pk<T>::pack(dl));
    }
    st_cs_v4(dx + i * V, Pk<T>::pack(acc));
  }
}

// ------------------------------------------------------------------------------ backward outputs

// Backward outputs from the adjoint state g and the saved h, one thread per
// (b, group, R rows, V columns), all D directions: dlam_k = g_k x, dx = sum_k g_k lam_k, and for the
// taps Da = g h_{t-1}[r-1], Db = g h_{t-1}[r], Dc = g h_{t-1}[r+1] (h_{-1} = 0, the neighbours along
// the scan-orthogonal axis) summed over the group's channels, then the normalisation Jacobian
// (gspn_common.cuh: jacobian). Coalesced along columns; the 3 h values per element come from a
// (V+2)-wide window of one row (vertical scans) or from three rows (horizontal scans; the next row's
// thread-iteration re-reads two of them from L1).
// V consecutive elements <-> floats through one 8- or 16-byte global access (read-only path for loads).
template <typename T, int V> struct GVec;
template <> struct GVec<__nv_bfloat16, 4> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float (&v)[4]) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
    v[0] = __uint_as_float(u.x << 16); v[1] = __uint_as_float(u.x & 0xFFFF0000u);
    v[2] = __uint_as_float(u.y << 16); v[3] = __uint_as_float(u.y & 0xFFFF0000u);
  }
  static __device__ __forceinline__ void store(__nv_bfloat16* p, const float (&v)[4]) {
    *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]));
  }
};
template <> struct GVec<float, 4> {
  static __device__ __forceinline__ void load(const float* p, float (&v)[4]) {
    const float4 u = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
  }
  static __device__ __forceinline__ void store(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};

template <typename T>
__device__ __forceinline__ float ldg_f(const T* p) { return to_f(__ldg(p)); }

// g * h_{t-1}[r-1], [r], [r+1] for V columns of row i of one chain, added to Da, Db, Dc.
template <typename T, int V>
__device__ __forceinline__ void accum_taps(uint32_t dir, const T* hp, int64_t H, int64_t W, int64_t i, int64_t j0,
                                           const float (&gv)[V], float (&Da)[V], float (&Db)[V], float (&Dc)[V]) {
  if (dir == GSPN_DIR_T2B || dir == GSPN_DIR_B2T) {
    // step t <-> row i; h_{t-1} is row i-1 (T2B) or i+1 (B2T); neighbours r+-1 = columns j+-1
    const int64_t ip = dir == GSPN_DIR_T2B ? i - 1 : i + 1;
    if (ip < 0 || ip >= H) return;
    const T* row = hp + ip * W;
    float v[V];
    GVec<T, V>::load(row + j0, v);
    const float lo = j0 > 0 ? ldg_f(row + j0 - 1) : 0.f;
    const float hi = j0 + V < W ? ldg_f(row + j0 + V) : 0.f;
#pragma unroll
    for (int q = 0; q < V; ++q) {
      Da[q] = fmaf(gv[q], q > 0 ? v[q - 1] : lo, Da[q]);
      Db[q] = fmaf(gv[q], v[q], Db[q]);
      Dc[q] = fmaf(gv[q], q + 1 < V ? v[q + 1] : hi, Dc[q]);
    }
  } else {
    // step t <-> column j; h_{t-1} is column j-1 (L2R) or j+1 (R2L); neighbours r+-1 = rows i+-1
    const bool l2r = dir == GSPN_DIR_L2R;
#pragma unroll
    for (int rr = 0; rr < 3; ++rr) {
      const int64_t ii = i - 1 + rr;
      if (ii < 0 || ii >= H) continue;
      const T* row = hp + ii * W;
      float v[V], sh[V];  // sh: h_{t-1} of row ii for the V columns
      GVec<T, V>::load(row + j0, v);
      if (l2r) {
        sh[0] = j0 > 0 ? ldg_f(row + j0 - 1) : 0.f;
#pragma unroll
        for (int q = 1; q < V; ++q) sh[q] = v[q - 1];
      } else {
#pragma unroll
        for (int q = 0; q + 1 < V; ++q) sh[q] = v[q + 1];
        sh[V - 1] = j0 + V < W ? ldg_f(row + j0 + V) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < V; ++q) {
        if (rr == 0) Da[q] = fmaf(gv[q], sh[q], Da[q]);
        else if (rr == 1) Db[q] = fmaf(gv[q], sh[q], Db[q]);
        else Dc[q] = fmaf(gv[q], sh[q], Dc[q]);
      }
    }
  }
}

// GSPN-local: the taps of a segment's first step act on a reset h_{t-1}, so their gradient is 0
// (the D terms of a7 vanish). Uniform branch, no cost for the global scan (kchunk = 0).
// One 32-bit modulo per call: a vertical direction's segment start depends on the row only, a horizontal
// one's on the column (bit q of reset_bits(j0, +1, ...) = column j0 + q starts a segment).
template <int V>
__device__ __forceinline__ void local_dw_mask(const ScanParams& p, uint32_t dir, int64_t i, int64_t j0, float (&ol)[V],
                                              float (&om)[V], float (&orr)[V]) {
  if (p.kchunk <= 0) return;
  const int k = static_cast<int>(p.kchunk);
  uint32_t m;
  if (dir == GSPN_DIR_T2B || dir == GSPN_DIR_B2T) {
    const int ii = static_cast<int>(i);
    const bool st = dir == GSPN_DIR_T2B ? ii % k == 0 : ((ii + 1) % k == 0 || ii == static_cast<int>(p.H) - 1);
    m = st ? 0xFFFFFFFFu : 0u;
  } else {
    const int jj = static_cast<int>(j0);
    m = reset_bits(jj, 1, dir == GSPN_DIR_L2R, k, V);
    if (dir == GSPN_DIR_R2L && static_cast<int>(p.W) - 1 - jj < V) m |= 1u << (static_cast<int>(p.W) - 1 - jj);
  }
#pragma unroll
  for (int q = 0; q < V; ++q)
    if ((m >> q) & 1u) ol[q] = om[q] = orr[q] = 0.f;
}

// dw_k for V columns of row i from the summed Da, Db, Dc.
template <typename T, int V>
__device__ __forceinline__ void finish_taps(const ScanParams& p, uint32_t dir, int64_t woff, int64_t i, int64_t j0,
                                            bool prenorm, const float (&Da)[V], const float (&Db)[V],
                                            const float (&Dc)[V]) {
  const bool vert = dir == GSPN_DIR_T2B || dir == GSPN_DIR_B2T;
  const int64_t P = vert ? p.W : p.H;
  float wl[V], wm[V], wr[V], ol[V], om[V], orr[V];
  GVec<T, V>::load(static_cast<const T*>(p.wl) + woff, wl);
  GVec<T, V>::load(static_cast<const T*>(p.wm) + woff, wm);
  GVec<T, V>::load(static_cast<const T*>(p.wr) + woff, wr);
#pragma unroll
  for (int q = 0; q < V; ++q) {
    const int64_t r = vert ? j0 + q : i;
    const bool hl = r >= 1, hr = r <= P - 2;
    jacobian<true>(wl[q], wm[q], wr[q], hl, hr, prenorm, hl ? Da[q] : 0.f, Db[q], hr ? Dc[q] : 0.f, ol[q], om[q], orr[q]);
  }
  local_dw_mask<V>(p, dir, i, j0, ol, om, orr);
  if (p.flags & GSPN_FLAG_DW_F32) {  // fp32 partial group sums (G < C only)
    for (int q = 0; q < V; ++q) {
      static_cast<float*>(p.dwl)[woff + q] = ol[q];
      static_cast<float*>(p.dwm)[woff + q] = om[q];
      static_cast<float*>(p.dwr)[woff + q] = orr[q];
    }
    return;
  }
  GVec<T, V>::store(static_cast<T*>(p.dwl) + woff, ol);
  GVec<T, V>::store(static_cast<T*>(p.dwm) + woff, om);
  GVec<T, V>::store(static_cast<T*>(p.dwr) + woff, orr);
}

template <typename T, int V, int R, bool kPerChannel>
__global__ void __launch_bounds__(256) bwd_out_kernel(ScanParams p, const T* __restrict__ g) {
  const int64_t W = p.W, H = p.H, HW = H * W;
  const int64_t nchunk = W / V, nrb = (H + R - 1) / R;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= p.B * p.G * nrb * nchunk) return;
  const int64_t j0 = (idx % nchunk) * V;
  const int64_t i0 = ((idx / nchunk) % nrb) * R;
  const int64_t bg = idx / (nchunk * nrb);
  const int64_t b = bg / p.G, grp = bg % p.G;
  const int64_t Cg = p.C / p.G;
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  const T* hbase = static_cast<const T*>(p.h);
  const T* xb = static_cast<const T*>(p.x);
  const T* lamb = static_cast<const T*>(p.lam);
  T* dlamb = static_cast<T*>(p.dlam);
  T* dxb = static_cast<T*>(p.dx);
  const int64_t iend = i0 + R < H ? i0 + R : H;
  for (int64_t i = i0; i < iend; ++i) {
    const int64_t rowoff = i * W + j0;
    if constexpr (kPerChannel) {
      const int64_t xoff = (b * p.C + grp) * HW + rowoff;
      float xv[V], dx[V];
      GVec<T, V>::load(xb + xoff, xv);
#pragma unroll
      for (int q = 0; q < V; ++q) dx[q] = 0.f;
      for (int k = 0; k < p.D; ++k) {
        const uint32_t dir = p.dirbit[k];
        const int64_t chain = (static_cast<int64_t>(k) * p.B + b) * p.C + grp;  // == weight plane (G = C)
        const int64_t off = chain * HW + rowoff;
        float gv[V], lv[V], dl[V], Da[V], Db[V], Dc[V];
        GVec<T, V>::load(g + off, gv);
        GVec<T, V>::load(lamb + off, lv);
#pragma unroll
        for (int q = 0; q < V; ++q) {
          dl[q] = gv[q] * xv[q];
          dx[q] = fmaf(gv[q], lv[q], dx[q]);
          Da[q] = Db[q] = Dc[q] = 0.f;
        }
        GVec<T, V>::store(dlamb + off, dl);
        accum_taps<T, V>(dir, hbase + chain * HW, H, W, i, j0, gv, Da, Db, Dc);
        finish_taps<T, V>(p, dir, off, i, j0, prenorm, Da, Db, Dc);
      }
      GVec<T, V>::store(dxb + xoff, dx);
    } else {
      float Da[4][V], Db[4][V], Dc[4][V];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int q = 0; q < V; ++q) Da[k][q] = Db[k][q] = Dc[k][q] = 0.f;
      for (int64_t cc = 0; cc < Cg; ++cc) {
        const int64_t c = grp * Cg + cc;
        const int64_t xoff = (b * p.C + c) * HW + rowoff;
        float xv[V], dx[V];
        GVec<T, V>::load(xb + xoff, xv);
#pragma unroll
        for (int q = 0; q < V; ++q) dx[q] = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k >= p.D) break;
          const int64_t chain = (static_cast<int64_t>(k) * p.B + b) * p.C + c;
          const int64_t off = chain * HW + rowoff;
          float gv[V], lv[V], dl[V];
          GVec<T, V>::load(g + off, gv);
          GVec<T, V>::load(lamb + off, lv);
#pragma unroll
          for (int q = 0; q < V; ++q) {
            dl[q] = gv[q] * xv[q];
            dx[q] = fmaf(gv[q], lv[q], dx[q]);
          }
          GVec<T, V>::store(dlamb + off, dl);
          accum_taps<T, V>(p.dirbit[k], hbase + chain * HW, H, W, i, j0, gv, Da[k], Db[k], Dc[k]);
        }
        GVec<T, V>::store(dxb + xoff, dx);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k >= p.D) break;
        const int64_t woff = ((static_cast<int64_t>(k) * p.B + b) * p.G + grp) * HW + rowoff;
        finish_taps<T, V>(p, p.dirbit[k], woff, i, j0, prenorm, Da[k], Db[k], Dc[k]);
      }
    }
  }
}

// V elements of T held packed in 32-bit words (loads issued early, unpacked at use).
template <typename T, int V>
struct PackedV {
  static constexpr int kWords = V * static_cast<int>(sizeof(T)) / 4;
  static_assert(kWords == 2 || kWords == 4, "8- or 16-byte vectors");
  uint32_t w[kWords];
  __device__ __forceinline__ void load(const T* p) {
    if constexpr (kWords == 4) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
      w[0] = u.x; w[1] = u.y; w[2] = u.z; w[3] = u.w;
    } else {
      const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
      w[0] = u.x; w[1] = u.y;
    }
  }
  __device__ __forceinline__ void unpack(float (&v)[V]) const {
#pragma unroll
    for (int i = 0; i < kWords; ++i) {
      if constexpr (sizeof(T) == 2) {
        v[2 * i] = __uint_as_float(w[i] << 16);
        v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
      } else {
        v[i] = __uint_as_float(w[i]);
      }
    }
  }
};

template <> struct GVec<float, 2> {
  static __device__ __forceinline__ void store(float* p, const float (&v)[2]) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  }
};

// Per-channel weights (G = C): one thread = (b, c, R rows, V columns), all D directions. Each row
// issues every load it needs (x; g, lam, w_l/m/r and the h_{t-1} window of every direction) before
// any arithmetic, so a thread has a whole row's worth of bytes in flight (the loop-carried version
// waited on ~4 dependent round trips per direction).
template <typename T, int V, int R, int kGrp>
__global__ void __launch_bounds__(256) bwd_out_pc_kernel(ScanParams p, const T* __restrict__ g) {
  const int64_t W = p.W, H = p.H, HW = H * W;
  const int64_t nchunk = W / V, nrb = (H + R - 1) / R;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= p.B * p.C * nrb * nchunk) return;
  const int64_t j0 = (idx % nchunk) * V;
  const int64_t i0 = ((idx / nchunk) % nrb) * R;
  const int64_t bc = idx / (nchunk * nrb);
  const int64_t b = bc / p.C, c = bc % p.C;
  const int D = p.D;
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  const T* hb = static_cast<const T*>(p.h);
  const T* lamb = static_cast<const T*>(p.lam);
  const T* wlb = static_cast<const T*>(p.wl);
  const T* wmb = static_cast<const T*>(p.wm);
  const T* wrb = static_cast<const T*>(p.wr);
  const int64_t iend = i0 + R < H ? i0 + R : H;
#pragma unroll 1
  for (int64_t i = i0; i < iend; ++i) {
    const int64_t rowoff = i * W + j0;
    PackedV<T, V> X;
    X.load(static_cast<const T*>(p.x) + bc * HW + rowoff);
    float xv[V], dx[V];
#pragma unroll
    for (int q = 0; q < V; ++q) dx[q] = 0.f;
#pragma unroll 1
    for (int k0 = 0; k0 < D; k0 += kGrp) {
    // ---- loads (kGrp directions)
    PackedV<T, V> Gk[kGrp], Lk[kGrp], WLk[kGrp], WMk[kGrp], WRk[kGrp], Hk[kGrp][3];
    float hs[kGrp][3];
#pragma unroll
    for (int kk = 0; kk < kGrp; ++kk) {
      const int k = k0 + kk;
      if (k >= D) break;
      const int64_t chain = (static_cast<int64_t>(k) * p.B + b) * p.C + c;  // == weight plane (G = C)
      const int64_t off = chain * HW + rowoff;
      Gk[kk].load(g + off);
      Lk[kk].load(lamb + off);
      WLk[kk].load(wlb + off);
      WMk[kk].load(wmb + off);
      WRk[kk].load(wrb + off);
      const uint32_t dir = p.dirbit[k];
      const T* hp = hb + chain * HW;
      if (dir == GSPN_DIR_T2B || dir == GSPN_DIR_B2T) {
        // h_{t-1} = row i-1 (T2B) / i+1 (B2T); neighbours r+-1 = columns j+-1
        int64_t ip = dir == GSPN_DIR_T2B ? i - 1 : i + 1;
        ip = ip < 0 ? 0 : (ip >= H ? H - 1 : ip);
        const T* row = hp + ip * W;
        Hk[kk][0].load(row + j0);
        hs[kk][0] = j0 > 0 ? ldg_f(row + j0 - 1) : 0.f;
        hs[kk][1] = j0 + V < W ? ldg_f(row + j0 + V) : 0.f;
      } else {
        // h_{t-1} = column j-1 (L2R) / j+1 (R2L); neighbours r+-1 = rows i+-1
        const int64_t col = dir == GSPN_DIR_L2R ? j0 - 1 : j0 + V;
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {
          int64_t ii = i - 1 + rr;
          ii = ii < 0 ? 0 : (ii >= H ? H - 1 : ii);
          const T* row = hp + ii * W;
          Hk[kk][rr].load(row + j0);
          hs[kk][rr] = (col >= 0 && col < W) ? ldg_f(row + col) : 0.f;
        }
      }
    }
    // ---- arithmetic + stores
    X.unpack(xv);
#pragma unroll
    for (int kk = 0; kk < kGrp; ++kk) {
      const int k = k0 + kk;
      if (k >= D) break;
      const int64_t chain = (static_cast<int64_t>(k) * p.B + b) * p.C + c;
      const int64_t off = chain * HW + rowoff;
      const uint32_t dir = p.dirbit[k];
      const bool vert = dir == GSPN_DIR_T2B || dir == GSPN_DIR_B2T;
      float gv[V], lv[V], dl[V], Da[V], Db[V], Dc[V];
      Gk[kk].unpack(gv);
      Lk[kk].unpack(lv);
#pragma unroll
      for (int q = 0; q < V; ++q) {
        dl[q] = gv[q] * xv[q];
        dx[q] = fmaf(gv[q], lv[q], dx[q]);
      }
      GVec<T, V>::store(static_cast<T*>(p.dlam) + off, dl);
      if (vert) {
        const int64_t ip = dir == GSPN_DIR_T2B ? i - 1 : i + 1;
        const bool ok = ip >= 0 && ip < H;
        float v[V];
        Hk[kk][0].unpack(v);
#pragma unroll
        for (int q = 0; q < V; ++q) {
          const float gq = ok ? gv[q] : 0.f;
          Da[q] = gq * (q > 0 ? v[q - 1] : hs[kk][0]);
          Db[q] = gq * v[q];
          Dc[q] = gq * (q + 1 < V ? v[q + 1] : hs[kk][1]);
        }
      } else {
        const bool l2r = dir == GSPN_DIR_L2R;
        float* Dr[3] = {Da, Db, Dc};
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {
          const int64_t ii = i - 1 + rr;
          const bool ok = ii >= 0 && ii < H;
          float v[V];
          Hk[kk][rr].unpack(v);
#pragma unroll
          for (int q = 0; q < V; ++q) {
            const float sh = l2r ? (q > 0 ? v[q - 1] : hs[kk][rr]) : (q + 1 < V ? v[q + 1] : hs[kk][rr]);
            Dr[rr][q] = ok ? gv[q] * sh : 0.f;
          }
        }
      }
      float wl[V], wm[V], wr[V], ol[V], om[V], orr[V];
      WLk[kk].unpack(wl);
      WMk[kk].unpack(wm);
      WRk[kk].unpack(wr);
      const int64_t P = vert ? W : H;
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const int64_t r = vert ? j0 + q : i;
        const bool hl = r >= 1, hr = r <= P - 2;
        jacobian<true>(wl[q], wm[q], wr[q], hl, hr, prenorm, hl ? Da[q] : 0.f, Db[q], hr ? Dc[q] : 0.f, ol[q], om[q],
                       orr[q]);
      }
      local_dw_mask<V>(p, dir, i, j0, ol, om, orr);
      GVec<T, V>::store(static_cast<T*>(p.dwl) + off, ol);
      GVec<T, V>::store(static_cast<T*>(p.dwm) + off, om);
      GVec<T, V>::store(static_cast<T*>(p.dwr) + off, orr);
    }
    }
    GVec<T, V>::store(static_cast<T*>(p.dx) + bc * HW + rowoff, dx);
  }
}

template <typename T, int V>
cudaError_t launch_out_pc(const ScanParams& p, const void* g, cudaStream_t s) {
  constexpr int R = 4;
  const int64_t n = p.B * p.C * ((p.H + R - 1) / R) * (p.W / V);
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  int grp = 2;  // directions whose loads are in flight together (experiments: GSPN_OUTK=1|2|4)
  if (const char* e = knob("GSPN_OUTK")) grp = atoi(e);
  const T* gt = static_cast<const T*>(g);
  if (grp == 1) bwd_out_pc_kernel<T, V, R, 1><<<blocks, 256, 0, s>>>(p, gt);
  else if (grp == 4) bwd_out_pc_kernel<T, V, R, 4><<<blocks, 256, 0, s>>>(p, gt);
  else bwd_out_pc_kernel<T, V, R, 2><<<blocks, 256, 0, s>>>(p, gt);
  return cudaGetLastError();
}

// ---- TMA-staged output kernel (G = C): a work unit is (b, c, RB image rows); the producer warp loads
// the unit's x, and per direction g, lam, w_l, w_m, w_r (RB rows) and h (RB + 2 rows: the halo rows
// i0-1 and i0+RB come from TMA, out-of-range rows as zero fill = h_{-1} = 0) into a shared-memory
// ring; 8 consumer warps compute from shared memory and store straight to global memory. Loads in
// flight no longer cost registers (the register-staged kernel was latency-bound at 2 CTAs/SM).
struct OutArgs {
  CUtensorMap x, g, lam, wl, wm, wr, h, dy;
  ScanParams p;
  int RB, BX, nbx, nstages, nrb;
  uint32_t box_rb, box_h;                            // bytes per TMA box (padded to 128)
  uint32_t tile_rb, tile_h, per_k, stage_bytes, tx;  // bytes
  uint32_t koff[4];                                  // byte offset of direction k's tiles in a stage
  uint32_t khoff[4];                                 // byte offset of direction k's h halo tile
  uint32_t dyoff;                                    // merged backward: the dy tile (after x)
  int64_t nunits;
  const unsigned* ready;                             // single launch: wait for D chains of the unit's plane
  int npack;
  // wide rows (W > 256, W % 256 == 0): 4D maps {256, W / 256, H, planes}, so ONE TMA box brings whole image
  // rows (the tile is [rows][W]) instead of W / 256 boxes per tensor; BX = W, nbx = 1 for the consumers
  int wide;
};

constexpr int kOutConsumers = 16;

// Rows [row, row + box rows) of one plane of an output-kernel tensor: box bx of a 3D map, or (wide) all of
// the row in one 4D box.
// kWide is a template parameter (a runtime branch here measured 13 % slower on config 2's output phase).
template <bool kWide>
__device__ __forceinline__ void out_load(const OutArgs& A, uint32_t dst, const CUtensorMap* map, int bx, int row,
                                         int plane, uint32_t bar, uint64_t pol) {
  if constexpr (kWide) tma_load4(dst, map, 0, 0, row, plane, bar, pol);
  else tma_load3(dst, map, bx * A.BX, row, plane, bar, pol);
}

// 4 consecutive elements at a shared-memory address (8- or 16-byte aligned).
template <typename T>
__device__ __forceinline__ void sm_ld4v(const uint8_t* p, float (&v)[4]) {
  if constexpr (sizeof(T) == 2) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    v[0] = __uint_as_float(u.x << 16); v[1] = __uint_as_float(u.x & 0xFFFF0000u);
    v[2] = __uint_as_float(u.y << 16); v[3] = __uint_as_float(u.y & 0xFFFF0000u);
  } else {
    const float4 u = *reinterpret_cast<const float4*>(p);
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
  }
}

// kVertDone: the fused recurrence already wrote dw of the vertical directions (hybrid backward): their
// w and h tiles are neither loaded nor used, only dlam and dx are formed for them.
// Body of the TMA-staged output kernel: warps [0, ncons) consume, warp ncons produces, any other warp
// returns at once. full[] / empty[] (A.nstages each, at the end of the ring) must be initialised with
// counts 1 / ncons. Shared by bwd_out_tma_kernel and the second phase of bwd_one_kernel.
template <typename T, bool kLocal, bool kVertDone, bool kMerged = false, bool kAllDone = false, bool kWide = false>
__device__ __forceinline__ void out_tma_body(const OutArgs& A, uint8_t* ring, uint64_t* full, uint64_t* empty,
                                             int ncons) {
  constexpr int V = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ScanParams& p = A.p;
  const int D = p.D, RB = A.RB, BX = A.BX;
  if (warp > ncons) return;
  if (warp == ncons) {  // producer
    if (lane == 0) {
      const uint64_t pol = policy_of(0);  // every input is read once
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = blockIdx.x; u < A.nunits; u += gridDim.x) {
        const uint32_t uq = static_cast<uint32_t>(u) / static_cast<uint32_t>(A.nrb);  // 32-bit: nunits < 2^31
        const int64_t bc = uq;
        const int i0 = static_cast<int>(static_cast<uint32_t>(u) - uq * static_cast<uint32_t>(A.nrb)) * RB;
        const int64_t b = bc / p.C, c = bc % p.C;
        mbar_wait_sleep(smem_u32(&empty[stage]), phase ^ 1);
        if (A.ready != nullptr) {  // every direction's g of this plane written (chains on other CTAs)
          const unsigned* r = A.ready + bc / A.npack;
          while (ld_acquire_gpu(r) < static_cast<unsigned>(D)) __nanosleep(128);
          fence_proxy_async_global();
        }
        const uint32_t fb = smem_u32(&full[stage]);
        mbar_arrive_tx(fb, A.tx);
        const uint32_t st = smem_u32(ring + static_cast<size_t>(stage) * A.stage_bytes);
        const uint32_t box_rb = A.box_rb, box_h = A.box_h;
        for (int bx = 0; bx < A.nbx; ++bx) out_load<kWide>(A, st + bx * box_rb, &A.x, bx, i0, static_cast<int>(bc), fb, pol);
        if constexpr (kMerged)
          for (int bx = 0; bx < A.nbx; ++bx)
            out_load<kWide>(A, st + A.dyoff + bx * box_rb, &A.dy, bx, i0, static_cast<int>(bc), fb, pol);
        for (int k = 0; k < D; ++k) {
          const int chain = static_cast<int>((static_cast<int64_t>(k) * p.B + b) * p.C + c);
          const uint32_t base = st + A.koff[k];
          const bool skip_w = kAllDone || (kVertDone && (p.dirbit[k] == GSPN_DIR_T2B || p.dirbit[k] == GSPN_DIR_B2T));
          for (int bx = 0; bx < A.nbx; ++bx) {
            out_load<kWide>(A, base + 0 * A.tile_rb + bx * box_rb, &A.g, bx, i0, chain, fb, pol);
            out_load<kWide>(A, base + 1 * A.tile_rb + bx * box_rb, &A.lam, bx, i0, chain, fb, pol);
            if (kMerged && skip_w)  // du = s h dy needs h at the pixel rows: the halo tile
              out_load<kWide>(A, st + A.khoff[k] + bx * A.box_h, &A.h, bx, i0 - 1, chain, fb, policy_of(1));
            if (skip_w) continue;
            out_load<kWide>(A, base + 2 * A.tile_rb + bx * box_rb, &A.wl, bx, i0, chain, fb, pol);
            out_load<kWide>(A, base + 3 * A.tile_rb + bx * box_rb, &A.wm, bx, i0, chain, fb, pol);
            out_load<kWide>(A, base + 4 * A.tile_rb + bx * box_rb, &A.wr, bx, i0, chain, fb, pol);
            out_load<kWide>(A, base + 5 * A.tile_rb + bx * box_h, &A.h, bx, i0 - 1, chain, fb, policy_of(1));
          }
        }
        if (++stage == A.nstages) { stage = 0; phase ^= 1; }
      }
    }
    return;
  }
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  const int64_t H = p.H, W = p.W, HW = H * W;
  const int64_t kstride = p.B * p.C * HW;  // between direction slabs of lam / g / h / w (G = C) / outputs
  const int nchunk = static_cast<int>(W / V);
  const int nthreads = ncons * 32;
  constexpr int es = static_cast<int>(sizeof(T));
  const uint32_t rowb = static_cast<uint32_t>(BX * es);  // bytes per box row
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t u = blockIdx.x; u < A.nunits; u += gridDim.x) {
    const uint32_t uq = static_cast<uint32_t>(u) / static_cast<uint32_t>(A.nrb);  // 32-bit: nunits < 2^31
    const int64_t bc = uq;
    const int i0 = static_cast<int>(static_cast<uint32_t>(u) - uq * static_cast<uint32_t>(A.nrb)) * RB;
    mbar_wait_sleep(smem_u32(&full[stage]), phase);
    const uint8_t* st = ring + static_cast<size_t>(stage) * A.stage_bytes;
    for (int idx = threadIdx.x; idx < RB * nchunk; idx += nthreads) {
      const int r = idx / nchunk;
      const int j0 = (idx - r * nchunk) * V;
      const int64_t i = i0 + r;
      if (i >= H) continue;
      // byte offsets of this chunk inside a [box][rows][BX] tile (computed once per chunk)
      const int bx = j0 >= BX ? j0 / BX : 0;
      const uint32_t col = static_cast<uint32_t>((j0 - bx * BX) * es);
      const uint32_t orb = bx * A.box_rb + r * rowb + col;     // RB-row tiles, row r
      const uint32_t oh = bx * A.box_h + r * rowb + col;       // halo tile, halo row r (= image row i-1)
      const bool has_lo = j0 > 0, has_hi = j0 + V < W;
      const uint32_t ohl = (j0 - bx * BX) > 0 ? oh - es : (bx - 1) * A.box_h + r * rowb + (BX - 1) * es;  // column j0-1
      const uint32_t ohh = (j0 - bx * BX) + V < BX ? oh + V * es : (bx + 1) * A.box_h + r * rowb;          // column j0+V
      const int64_t off0 = bc * HW + i * W + j0;  // x / dx; direction k adds k * kstride (chain k, b, c)
      float xv[V], dx[V], dyv[V];
      sm_ld4v<T>(st + orb, xv);
      if constexpr (kMerged) sm_ld4v<T>(st + A.dyoff + orb, dyv);
#pragma unroll
      for (int q = 0; q < V; ++q) dx[q] = 0.f;
      for (int k = 0; k < D; ++k) {
        const uint8_t* base = st + A.koff[k];
        const uint8_t* ht = st + A.khoff[k];
        const uint32_t dir = p.dirbit[k];
        const bool vert = dir == GSPN_DIR_T2B || dir == GSPN_DIR_B2T;
        const int64_t off = off0 + k * kstride;
        float gv[V], lv[V], dl[V], Da[V], Db[V], Dc[V];
        sm_ld4v<T>(base + orb, gv);
        sm_ld4v<T>(base + A.tile_rb + orb, lv);
#pragma unroll
        for (int q = 0; q < V; ++q) {
          dl[q] = gv[q] * xv[q];
          dx[q] = fmaf(gv[q], lv[q], dx[q]);
        }
        GVec<T, V>::store(static_cast<T*>(p.dlam) + off, dl);
        if constexpr (kMerged) {  // du_k = s h_k dy: h at image row i = halo row r + 1
          float hv[V], du[V];
          sm_ld4v<T>(ht + oh + rowb, hv);
#pragma unroll
          for (int q = 0; q < V; ++q) du[q] = p.merge_scale * hv[q] * dyv[q];
          GVec<T, V>::store(static_cast<T*>(p.du) + off, du);
        }
        if ((kVertDone && vert) || kAllDone) continue;
        if (vert) {
          // h_{t-1}: image row i-1 (T2B) / i+1 (B2T) = halo row r / r+2; neighbours = columns j+-1
          const uint32_t ro = dir == GSPN_DIR_T2B ? 0u : 2u * rowb;
          float v[V];
          sm_ld4v<T>(ht + oh + ro, v);
          const float lo = has_lo ? to_f(*reinterpret_cast<const T*>(ht + ohl + ro)) : 0.f;
          const float hi = has_hi ? to_f(*reinterpret_cast<const T*>(ht + ohh + ro)) : 0.f;
#pragma unroll
          for (int q = 0; q < V; ++q) {
            Da[q] = gv[q] * (q > 0 ? v[q - 1] : lo);
            Db[q] = gv[q] * v[q];
            Dc[q] = gv[q] * (q + 1 < V ? v[q + 1] : hi);
          }
        } else {
          // h_{t-1}: column j-1 (L2R) / j+1 (R2L); neighbours = image rows i-1, i, i+1 = halo rows r..r+2
          const bool l2r = dir == GSPN_DIR_L2R;
          const bool e_ok = l2r ? has_lo : has_hi;
          const uint32_t oe = l2r ? ohl : ohh;
          float* Dr[3] = {Da, Db, Dc};
#pragma unroll
          for (int rr = 0; rr < 3; ++rr) {
            float v[V];
            sm_ld4v<T>(ht + oh + rr * rowb, v);
            const float e = e_ok ? to_f(*reinterpret_cast<const T*>(ht + oe + rr * rowb)) : 0.f;
#pragma unroll
            for (int q = 0; q < V; ++q) {
              const float sh = l2r ? (q > 0 ? v[q - 1] : e) : (q + 1 < V ? v[q + 1] : e);
              Dr[rr][q] = gv[q] * sh;
            }
          }
        }
        float wl[V], wm[V], wr[V], ol[V], om[V], orr[V];
        sm_ld4v<T>(base + 2 * A.tile_rb + orb, wl);
        sm_ld4v<T>(base + 3 * A.tile_rb + orb, wm);
        sm_ld4v<T>(base + 4 * A.tile_rb + orb, wr);
        if (vert) {
#pragma unroll
          for (int q = 0; q < V; ++q) {
            const bool hl = j0 + q >= 1, hr = j0 + q <= W - 2;
            jacobian<true>(wl[q], wm[q], wr[q], hl, hr, prenorm, Da[q], Db[q], Dc[q], ol[q], om[q], orr[q]);
          }
        } else {
          const bool hl = i >= 1, hr = i <= H - 2;
#pragma unroll
          for (int q = 0; q < V; ++q)
            jacobian<true>(wl[q], wm[q], wr[q], hl, hr, prenorm, Da[q], Db[q], Dc[q], ol[q], om[q], orr[q]);
        }
        if constexpr (kLocal) local_dw_mask<V>(p, dir, i, j0, ol, om, orr);
        GVec<T, V>::store(static_cast<T*>(p.dwl) + off, ol);
        GVec<T, V>::store(static_cast<T*>(p.dwm) + off, om);
        GVec<T, V>::store(static_cast<T*>(p.dwr) + off, orr);
      }
      GVec<T, V>::store(static_cast<T*>(p.dx) + off0, dx);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&empty[stage]));
    if (++stage == A.nstages) { stage = 0; phase ^= 1; }
  }
}

template <typename T, bool kLocal, bool kVertDone>
__global__ void __launch_bounds__((kOutConsumers + 1) * 32, 1) bwd_out_tma_kernel(const __grid_constant__ OutArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(A.nstages) * A.stage_bytes);
  uint64_t* empty = full + A.nstages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < A.nstages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), kOutConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  out_tma_body<T, kLocal, kVertDone>(A, ring, full, empty, kOutConsumers);
}

// ---- Single-launch backward (north_star "one persistent kernel per call"; "Kernel Fuse";
// SURVEY.md §8(c) reading 17). One cooperative persistent launch: phase 1 is the fused adjoint recurrence
// (bwd_fused_body: g, and dw of the vertical chains), then a grid-wide barrier (every g must be complete
// before any (b, c, rows) unit sums dx over the directions), then phase 2 is the TMA-staged output pass
// (out_tma_body: dlam, dx, and dw of the horizontal chains) on the same CTAs, their shared memory re-carved
// as the output ring. Phase 2's consumers are phase 1's consumer warps, its producer phase 1's producer.
struct OneArgs {
  StreamArgs s;
  OutArgs o;
};

__device__ __forceinline__ void mbar_inval(uint32_t bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
template <typename T, int kPre, bool kLocal, bool kMerged = false, bool kHF = false, bool kWide = false>
__global__ void __launch_bounds__((kMaxNWC + 2) * 32, 1) bwd_one_kernel(const __grid_constant__ OneArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Plan& pl = A.s.plan;
  const Smem m = carve(smem_raw, pl);
  // plane-readiness counters start at 0 before any chain can finish
  if (A.s.ready != nullptr) {
    const int64_t npl = (pl.nbc + pl.npack - 1) / pl.npack;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < npl;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
      A.s.ready[i] = 0u;
    __threadfence();
  }
  init_barriers<false>(m, pl);
  if (A.s.ready != nullptr) cooperative_groups::this_grid().sync();  // counters zeroed before any chain ends
  bwd_fused_body<T, kPre, kLocal, kMerged, kHF>(A.s, m);
  // Grid-wide barrier between the phases (default). With readiness counters (experiments: GSPN_PLANE_READY)
  // a unit's producer instead waits until the D chains of its plane have published their g (storer:
  // completed stores, gpu-scope fence, counter), so CTAs that finish phase 1 early start phase 2.
  fence_proxy_async_global();
  __syncthreads();
  if (A.s.ready == nullptr) cooperative_groups::this_grid().sync();
  const OutArgs& O = A.o;
  uint64_t* full = reinterpret_cast<uint64_t*>(m.ring + static_cast<size_t>(O.nstages) * O.stage_bytes);
  uint64_t* empty = full + O.nstages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < pl.nstages; ++s) {
      mbar_inval(smem_u32(&m.full[s]));
      mbar_inval(smem_u32(&m.empty[s]));
      mbar_inval(smem_u32(&m.done[s]));
    }
    for (int i = 0; i < 4; ++i) mbar_inval(smem_u32(&m.xb[i]));
    for (int s = 0; s < O.nstages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), pl.nwc);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();        // phase-1 generic writes of the ring before phase-2 TMA writes into it
  fence_proxy_async_global();
  __syncthreads();
  out_tma_body<T, kLocal, true, kMerged, kHF, kWide>(O, m.ring, full, empty, pl.nwc);
}

// ---- Recompute-h backward in one launch (NEXT-3): bwd_rc_body (adjoint + tap gradients of both
// orientations, h recomputed per half-tile from the forward's checkpoints) | grid barrier | dlam and dx.
template <typename T, int kPre>
__global__ void __launch_bounds__((kMaxNWC + 2) * 32, 1) bwd_rc_kernel(const __grid_constant__ OneArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Plan& pl = A.s.plan;
  const Smem m = carve(smem_raw, pl);
  init_barriers<false>(m, pl);
  bwd_rc_body<T, kPre>(A.s, m);
  fence_proxy_async_global();
  __syncthreads();
  cooperative_groups::this_grid().sync();
  const OutArgs& O = A.o;
  uint64_t* full = reinterpret_cast<uint64_t*>(m.ring + static_cast<size_t>(O.nstages) * O.stage_bytes);
  uint64_t* empty = full + O.nstages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < pl.nstages; ++s) {
      mbar_inval(smem_u32(&m.full[s]));
      mbar_inval(smem_u32(&m.empty[s]));
      mbar_inval(smem_u32(&m.done[s]));
    }
    for (int i = 0; i < 4; ++i) mbar_inval(smem_u32(&m.xb[i]));
    for (int s = 0; s < O.nstages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), pl.nwc);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();
  fence_proxy_async_global();
  __syncthreads();
  out_tma_body<T, false, true, false, true>(O, m.ring, full, empty, pl.nwc);
}

// ---- Forward through the output gate + direction merge in one launch (NEXT-1, Eq. 2):
// phase 1 is the forward scan (h to the caller's buffer or the workspace), then a grid-wide barrier, then
// phase 2 forms y = s sum_d u_d (.) h_d over [B, C, H, W] on the same CTAs (16-byte vectors, grid-stride).
struct OneFwdArgs {
  StreamArgs s;
  const void* u;
  void* y;
  float scale;
  int64_t N;  // B C H W (a multiple of the vector width)
};

template <typename T, int kPre, bool kLocal>
__global__ void __launch_bounds__((kMaxNWC + 2) * 32, 1) fwd_one_kernel(const __grid_constant__ OneFwdArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Smem m = carve(smem_raw, A.s.plan);
  init_barriers<false>(m, A.s.plan);
  fwd_stream_body<T, kPre, false, kLocal>(A.s, m);
  fence_proxy_async_global();  // h: generic stores (vertical) and completed TMA stores (horizontal)
  __syncthreads();
  cooperative_groups::this_grid().sync();
  constexpr int V = 16 / static_cast<int>(sizeof(T));
  const int D = static_cast<int>(A.s.p.D);
  const T* h = static_cast<const T*>(A.s.p.hout);
  const T* u = static_cast<const T*>(A.u);
  T* y = static_cast<T*>(A.y);
  const int64_t nv = A.N / V;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint4 hq[4], uq[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      if (d >= D) break;
      hq[d] = __ldcg(reinterpret_cast<const uint4*>(h + d * A.N + i * V));  // written by this launch: not .nc
      uq[d] = ld_nc_v4(u + d * A.N + i * V);
    }
    float acc[V];
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] = 0.f;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      if (d >= D) break;
#pragma unroll
      for (int e = 0; e < V; ++e) acc[e] = fmaf(hget<T>(uq[d], e), hget<T>(hq[d], e), acc[e]);
    }
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] *= A.scale;
    st_cs_v4(y + i * V, Pk<T>::pack(acc));
  }
}

// ---- Grouped weights (G < C): a unit is (b, group, RB rows); the ring streams one channel of the
// group per stage (x, and per direction g, lam and the h halo tile), every thread keeps the group sums
// Da/Db/Dc of its 4-column chunk for all directions in registers, and after the group's last channel
// reads w from global memory once and writes dw. One chunk per consumer thread (RB W / 4 <= 512).
template <typename T, bool kLocal, bool kWide = false>
__global__ void __launch_bounds__((kOutConsumers + 1) * 32, 1) bwd_out_grp_tma_kernel(const __grid_constant__ OutArgs A) {
  constexpr int V = 4;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(A.nstages) * A.stage_bytes);
  uint64_t* empty = full + A.nstages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ScanParams& p = A.p;
  const int D = p.D, RB = A.RB, BX = A.BX;
  const int64_t Cg = p.C / p.G;
  if (threadIdx.x == 0) {
    for (int s = 0; s < A.nstages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), kOutConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kOutConsumers) {  // producer
    if (lane == 0) {
      const uint64_t pol = policy_of(0);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = blockIdx.x; u < A.nunits; u += gridDim.x) {
        const uint32_t uq = static_cast<uint32_t>(u) / static_cast<uint32_t>(A.nrb);  // 32-bit: nunits < 2^31
        const int64_t bg = uq;
        const int i0 = static_cast<int>(static_cast<uint32_t>(u) - uq * static_cast<uint32_t>(A.nrb)) * RB;
        const int64_t b = bg / p.G, grp = bg % p.G;
        for (int64_t cc = 0; cc < Cg; ++cc) {
          const int64_t bc = b * p.C + grp * Cg + cc;
          mbar_wait_sleep(smem_u32(&empty[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full[stage]);
          mbar_arrive_tx(fb, A.tx);
          const uint32_t st = smem_u32(ring + static_cast<size_t>(stage) * A.stage_bytes);
          for (int bx = 0; bx < A.nbx; ++bx) out_load<kWide>(A, st + bx * A.box_rb, &A.x, bx, i0, static_cast<int>(bc), fb, pol);
          for (int k = 0; k < D; ++k) {
            const int chain = static_cast<int>(static_cast<int64_t>(k) * p.B * p.C + bc);
            const uint32_t base = st + A.tile_rb + k * A.per_k;
            for (int bx = 0; bx < A.nbx; ++bx) {
              out_load<kWide>(A, base + bx * A.box_rb, &A.g, bx, i0, chain, fb, pol);
              out_load<kWide>(A, base + A.tile_rb + bx * A.box_rb, &A.lam, bx, i0, chain, fb, pol);
              out_load<kWide>(A, base + 2 * A.tile_rb + bx * A.box_h, &A.h, bx, i0 - 1, chain, fb, policy_of(1));
            }
          }
          if (++stage == A.nstages) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  const int64_t H = p.H, W = p.W, HW = H * W;
  const int64_t kstride = p.B * p.C * HW;   // direction slabs of lam / g / h / dlam
  const int64_t kwstride = p.B * p.G * HW;  // direction slabs of w / dw
  const bool dw_f32 = (p.flags & GSPN_FLAG_DW_F32) != 0;
  const int nchunk = static_cast<int>(W / V);
  constexpr int es = static_cast<int>(sizeof(T));
  const uint32_t rowb = static_cast<uint32_t>(BX * es);
  const int idx = threadIdx.x;  // this thread's chunk (one per thread)
  const int r = idx / nchunk;
  const int j0 = (idx - r * nchunk) * V;
  const int bx = j0 >= BX ? j0 / BX : 0;
  const uint32_t col = static_cast<uint32_t>((j0 - bx * BX) * es);
  const uint32_t orb = bx * A.box_rb + r * rowb + col;
  const uint32_t oh = bx * A.box_h + r * rowb + col;
  const bool has_lo = j0 > 0, has_hi = j0 + V < W;
  const uint32_t ohl = (j0 - bx * BX) > 0 ? oh - es : (bx - 1) * A.box_h + r * rowb + (BX - 1) * es;
  const uint32_t ohh = (j0 - bx * BX) + V < BX ? oh + V * es : (bx + 1) * A.box_h + r * rowb;
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t u = blockIdx.x; u < A.nunits; u += gridDim.x) {
    const uint32_t uq = static_cast<uint32_t>(u) / static_cast<uint32_t>(A.nrb);  // 32-bit: nunits < 2^31
    const int64_t bg = uq;
    const int i0 = static_cast<int>(static_cast<uint32_t>(u) - uq * static_cast<uint32_t>(A.nrb)) * RB;
    const int64_t b = bg / p.G, grp = bg % p.G;
    const int64_t i = i0 + r;
    const bool valid = r < RB && i < H;
    float Da[4][V], Db[4][V], Dc[4][V];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int q = 0; q < V; ++q) Da[k][q] = Db[k][q] = Dc[k][q] = 0.f;
    for (int64_t cc = 0; cc < Cg; ++cc) {
      mbar_wait_sleep(smem_u32(&full[stage]), phase);
      const uint8_t* st = ring + static_cast<size_t>(stage) * A.stage_bytes;
      if (valid) {
        const int64_t bc = b * p.C + grp * Cg + cc;
        const int64_t off0 = bc * HW + i * W + j0;
        float xv[V], dx[V];
        sm_ld4v<T>(st + orb, xv);
#pragma unroll
        for (int q = 0; q < V; ++q) dx[q] = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k >= D) break;
          const uint8_t* base = st + A.tile_rb + k * A.per_k;
          const uint8_t* ht = base + 2 * A.tile_rb;
          const uint32_t dir = p.dirbit[k];
          const int64_t off = off0 + k * kstride;
          float gv[V], lv[V], dl[V];
          sm_ld4v<T>(base + orb, gv);
          sm_ld4v<T>(base + A.tile_rb + orb, lv);
#pragma unroll
          for (int q = 0; q < V; ++q) {
            dl[q] = gv[q] * xv[q];
            dx[q] = fmaf(gv[q], lv[q], dx[q]);
          }
          GVec<T, V>::store(static_cast<T*>(p.dlam) + off, dl);
          if (dir == GSPN_DIR_T2B || dir == GSPN_DIR_B2T) {
            const uint32_t ro = dir == GSPN_DIR_T2B ? 0u : 2u * rowb;
            float v[V];
            sm_ld4v<T>(ht + oh + ro, v);
            const float lo = has_lo ? to_f(*reinterpret_cast<const T*>(ht + ohl + ro)) : 0.f;
            const float hi = has_hi ? to_f(*reinterpret_cast<const T*>(ht + ohh + ro)) : 0.f;
#pragma unroll
            for (int q = 0; q < V; ++q) {
              Da[k][q] = fmaf(gv[q], q > 0 ? v[q - 1] : lo, Da[k][q]);
              Db[k][q] = fmaf(gv[q], v[q], Db[k][q]);
              Dc[k][q] = fmaf(gv[q], q + 1 < V ? v[q + 1] : hi, Dc[k][q]);
            }
          } else {
            const bool l2r = dir == GSPN_DIR_L2R;
            const bool e_ok = l2r ? has_lo : has_hi;
            const uint32_t oe = l2r ? ohl : ohh;
#pragma unroll
            for (int rr = 0; rr < 3; ++rr) {
              float v[V];
              sm_ld4v<T>(ht + oh + rr * rowb, v);
              const float e = e_ok ? to_f(*reinterpret_cast<const T*>(ht + oe + rr * rowb)) : 0.f;
#pragma unroll
              for (int q = 0; q < V; ++q) {
                const float sh = l2r ? (q > 0 ? v[q - 1] : e) : (q + 1 < V ? v[q + 1] : e);
                if (rr == 0) Da[k][q] = fmaf(gv[q], sh, Da[k][q]);
                else if (rr == 1) Db[k][q] = fmaf(gv[q], sh, Db[k][q]);
                else Dc[k][q] = fmaf(gv[q], sh, Dc[k][q]);
              }
            }
          }
        }
        GVec<T, V>::store(static_cast<T*>(p.dx) + off0, dx);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[stage]));
      if (++stage == A.nstages) { stage = 0; phase ^= 1; }
    }
    if (valid) {
      const int64_t woff0 = (b * p.G + grp) * HW + i * W + j0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k >= D) break;
        const uint32_t dir = p.dirbit[k];
        const bool vert = dir == GSPN_DIR_T2B || dir == GSPN_DIR_B2T;
        const int64_t woff = woff0 + k * kwstride;
        float wl[V], wm[V], wr[V], ol[V], om[V], orr[V];
        GVec<T, V>::load(static_cast<const T*>(p.wl) + woff, wl);
        GVec<T, V>::load(static_cast<const T*>(p.wm) + woff, wm);
        GVec<T, V>::load(static_cast<const T*>(p.wr) + woff, wr);
#pragma unroll
        for (int q = 0; q < V; ++q) {
          const int64_t rp = vert ? j0 + q : i;
          const int64_t P = vert ? W : H;
          jacobian<true>(wl[q], wm[q], wr[q], rp >= 1, rp <= P - 2, prenorm, Da[k][q], Db[k][q], Dc[k][q], ol[q],
                         om[q], orr[q]);
        }
        if constexpr (kLocal) local_dw_mask<V>(p, dir, i, j0, ol, om, orr);
        if (dw_f32) {  // fp32 partial group sums (GSPN_FLAG_DW_F32: reduced across devices in fp32)
          GVec<float, V>::store(static_cast<float*>(p.dwl) + woff, ol);
          GVec<float, V>::store(static_cast<float*>(p.dwm) + woff, om);
          GVec<float, V>::store(static_cast<float*>(p.dwr) + woff, orr);
        } else {
          GVec<T, V>::store(static_cast<T*>(p.dwl) + woff, ol);
          GVec<T, V>::store(static_cast<T*>(p.dwm) + woff, om);
          GVec<T, V>::store(static_cast<T*>(p.dwr) + woff, orr);
        }
      }
    }
  }
}

template <typename T, int V, bool kPerChannel>
cudaError_t launch_out(const ScanParams& p, const void* g, cudaStream_t s) {
  constexpr int R = 8;
  const int64_t n = p.B * p.G * ((p.H + R - 1) / R) * (p.W / V);
  const int64_t blocks = (n + 255) / 256;
  bwd_out_kernel<T, V, R, kPerChannel><<<static_cast<unsigned>(blocks), 256, 0, s>>>(p, static_cast<const T*>(g));
  return cudaGetLastError();
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

// 3D map over a [planes][H][W] tensor. plane_mid: dims ordered (W, planes, H) instead of (W, H, planes)
// (packed vertical tiles: one box = K rows of npack consecutive planes, step-major in shared memory).
// L2 promotion of the swizzled (horizontal-tile) maps: experiments only, GSPN_L2PROMO = 64 | 128 | 256.
CUtensorMapL2promotion horiz_promotion() {
  const char* e = knob("GSPN_L2PROMO");
  const int v = e ? atoi(e) : 0;
  return v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
         : v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
}

bool encode(CUtensorMap* m, const void* base, gspn_dtype_t dt, int64_t W, int64_t H, int64_t planes, int box0,
            int box1, bool swizzle32, int box2 = 1, bool plane_mid = false) {
  auto fn = get_encode();
  if (!fn) return false;
  const size_t s = dt == GSPN_BF16 ? 2 : 4;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(planes)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(W * s), static_cast<cuuint64_t>(W * H * s)};
  if (plane_mid) {
    dims[1] = static_cast<cuuint64_t>(planes);
    dims[2] = static_cast<cuuint64_t>(H);
    strides[0] = static_cast<cuuint64_t>(W * H * s);
    strides[1] = static_cast<cuuint64_t>(W * s);
  }
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box0), static_cast<cuuint32_t>(box1), static_cast<cuuint32_t>(box2)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, dt == GSPN_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  swizzle32 ? horiz_promotion() : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Output-kernel maps: 3D {W, H, planes} with box {bx, rows, 1}, or (wide) 4D {256, W / 256, H, planes} with box
// {256, W / 256, rows, 1}: whole rows in one box, landing as [rows][W].
bool encode_rows(CUtensorMap* m, const void* base, gspn_dtype_t dt, int64_t W, int64_t H, int64_t planes, int bx,
                 int rows, bool wide) {
  if (!wide) return encode(m, base, dt, W, H, planes, bx, rows, false);
  auto fn = get_encode();
  if (!fn) return false;
  const size_t s = dt == GSPN_BF16 ? 2 : 4;
  cuuint64_t dims[4] = {256u, static_cast<cuuint64_t>(W / 256), static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(planes)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(256 * s), static_cast<cuuint64_t>(W * s), static_cast<cuuint64_t>(W * H * s)};
  cuuint32_t box[4] = {256u, static_cast<cuuint32_t>(W / 256), static_cast<cuuint32_t>(rows), 1u};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, dt == GSPN_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int sm_count() { return device_sm_count(); }
int smem_optin() { return device_smem_optin(); }

constexpr int kSmemTail = 26624;  // mbarriers (3 per stage), exchange rows (3 x 2 x 16 x 64 floats = 24 KB), cluster edges

// Shape eligibility + plan (nin: tensors per tile).
bool make_plan(const ScanParams& p, gspn_dtype_t dt, int nin, Plan* pl) {
  const int s = dt == GSPN_BF16 ? 2 : 4;
  // TMA: 16-byte aligned row stride; the horizontal 16-byte chunks tile W exactly
  if ((p.W * s) % 16 != 0) return false;
  bool any_v = false, any_h = false;
  for (int k = 0; k < p.D; ++k) {
    if (p.dirbit[k] == GSPN_DIR_T2B || p.dirbit[k] == GSPN_DIR_B2T) any_v = true; else any_h = true;
  }
  const int64_t maxP = std::max<int64_t>(any_v ? p.W : 0, any_h ? p.H : 0);
  memset(pl, 0, sizeof *pl);
  pl->K = 32 / s;
  const int GH = pl->K / 2;
  pl->E = 2;
  pl->es = s;
  pl->own = 64 - 2 * GH;
  pl->cl = 1;
  pl->nwc = static_cast<int>((maxP + pl->own - 1) / pl->own);  // warp w owns [w own, (w+1) own)
  // positions any lane reads (clamped to the tile); the TMA boxes cover them so no lane reads stale rows
  int cover = static_cast<int>(std::min<int64_t>(kPpad, (pl->nwc - 1) * pl->own - GH + 64));
  const bool force_split = (p.flags & GSPN_FLAG_FORCE_SPLIT) != 0;
  if (pl->nwc > 11 || force_split) {
    // P-split over a cluster: each CTA owns the positions its warps own while their ghosts stay
    // inside its 512-position tile (10 x 48 bf16 / 9 x 56 fp32). GSPN_FLAG_FORCE_SPLIT (tests): at
    // least 2 CTAs per chain, so the cluster path can be checked bitwise against the unsplit one.
    int nwc_c = (kPpad - 2 * GH) / pl->own;
    if (const char* e = knob("GSPN_CL_NWC")) nwc_c = std::max(1, std::min(nwc_c, atoi(e)));  // experiments
    if (force_split) {
      const int64_t half = (maxP + 1) / 2;
      nwc_c = std::max(1, std::min<int>(nwc_c, static_cast<int>((half + pl->own - 1) / pl->own)));
    }
    pl->ownc = nwc_c * pl->own;
    pl->cl = static_cast<int>((maxP + pl->ownc - 1) / pl->ownc);
    if (pl->cl > 8 || knob("GSPN_NOCLUSTER")) return false;
    pl->nwc = nwc_c;
    cover = kPpad;
    pl->bhs = pl->ownc / 2;  // <= 256 rows per TMA store box
    pl->nbhs = 2;
  }
  pl->ppad = kPpad;
  pl->bw = kRowB / s;
  pl->nbw = (cover + pl->bw - 1) / pl->bw;
  int bh = 8;
  while (bh < cover && bh < 256) bh <<= 1;
  pl->bh = bh;
  pl->nbh = (cover + bh - 1) / bh;
  pl->nin = nin;
  pl->tile_bytes = kTile;
  pl->stage_bytes = nin * kTile;
  pl->tx_v = static_cast<uint32_t>(nin * pl->nbw * pl->bw * pl->K * s);
  pl->tx_h = static_cast<uint32_t>(nin * pl->nbh * pl->bh * 32);
  pl->npack = 1;
  pl->nbc = p.B * p.C;
  pl->vstep = kRowB;
  const int64_t PH = std::max<int64_t>(p.H, p.W);  // packing needs both orientations to fit
  if (pl->cl == 1 && p.G == p.C && PH <= kPpad / 2 && pl->nbc > 1 && !knob("GSPN_NOPACK")) {
    // a divisor of B C: no partial pack, so a packed TMA store never spills into the next direction
    int np = static_cast<int>(std::min<int64_t>({kPpad / PH, 256, pl->nbc}));
    while (pl->nbc % np != 0) --np;
    if (np >= 2) {
      pl->npack = np;
      pl->vstep = static_cast<uint32_t>(np * p.W * s);
      pl->nwc = static_cast<int>((np * PH + pl->own - 1) / pl->own);
      if (pl->nwc > 11) return false;
      pl->tx_v = static_cast<uint32_t>(nin * np * p.W * pl->K * s);
      pl->tx_h = static_cast<uint32_t>(nin * np * p.H * 32);
    }
  }
  const int budget = smem_optin() - 1024 /*alignment*/ - kSmemTail;
  int ns = budget / static_cast<int>(pl->stage_bytes);
  if (ns > 6) ns = 6;
  if (const char* e = knob("GSPN_NSTAGES")) ns = std::max(1, std::min(ns, atoi(e)));  // experiments
  if (ns < 1 || (ns < 2 && !knob("GSPN_NSTAGES"))) return false;
  pl->nstages = ns;
  pl->nchains = p.D * ((pl->nbc + pl->npack - 1) / pl->npack);  // work items: packs of chains
  if (pl->nchains >= (int64_t{1} << 31) || pl->nbc >= (int64_t{1} << 31)) return false;  // 32-bit make_chain
  // GSPN-local (kchunk > 0): each segment is an independent work item when segment boundaries fall on tile
  // boundaries in scan order (kchunk, H and W multiples of K): more, shorter items for the persistent grid,
  // bitwise the same arithmetic (a segment starts from h = 0 / g = 0 either way)
  pl->nseg = 1;
  pl->kt = 0;
  if (p.kchunk > 0 && p.kchunk % pl->K == 0 && p.H % pl->K == 0 && p.W % pl->K == 0 && !knob("GSPN_NO_SEGITEMS") &&
      !knob("GSPN_PLANE_READY")) {
    const int64_t Lmax = std::max<int64_t>(p.H, p.W);
    pl->nseg = static_cast<int>((Lmax + p.kchunk - 1) / p.kchunk);
    pl->kt = static_cast<int>(p.kchunk / pl->K);
    if (pl->nchains * pl->nseg < (int64_t{1} << 31)) pl->nchains *= pl->nseg;
    else pl->nseg = 1;
  }
  pl->smem_bytes = 1024 + ns * pl->stage_bytes + kSmemTail;
  // L2 priorities (experiments: GSPN_POL="x,vin,hin,vout,hout,acc", each 0|1|2)
  // horizontal loads evict_last: +0.5 % (same-box A/B x3); x (read by the plane's 4 directions) evict_last:
  // forward DRAM reads 12.20 -> 12.12 GB and 2.788 -> 2.779 ms (ncu, 2 launches each)
  static const int def_pol[6] = {2, 0, 2, 0, 1, 1};
  for (int i = 0; i < 6; ++i) pl->pol[i] = def_pol[i];
  if (const char* e = knob("GSPN_POL")) {
    int v[6], n = sscanf(e, "%d,%d,%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3], &v[4], &v[5]);
    for (int i = 0; i < n && i < 6; ++i) pl->pol[i] = v[i];
  }
  if (const char* e = knob("GSPN_NULL")) pl->null_compute = atoi(e) != 0;
  return true;
}

// ins: tensors per tile; outs: horizontal output tensors stored by the storer (same box as inputs).
bool fill_maps(StreamArgs* A, const void* const* ins, int nin, void* const* outs, const int64_t* in_planes,
               int64_t out_planes, int nout, gspn_dtype_t dt) {
  const Plan& pl = A->plan;
  const ScanParams& p = A->p;
  if (pl.npack > 1) {
    for (int t = 0; t < nin; ++t) {
      if (!encode(&A->in[0][t], ins[t], dt, p.W, p.H, in_planes[t], p.W, pl.npack, false, pl.K, true)) return false;
      if (!encode(&A->in[1][t], ins[t], dt, p.W, p.H, in_planes[t], pl.K, p.H, true, pl.npack)) return false;
    }
    for (int t = 0; t < nout; ++t)
      if (!encode(&A->out[1][t], outs[t], dt, p.W, p.H, out_planes, pl.K, p.H, true, pl.npack)) return false;
    return true;
  }
  for (int t = 0; t < nin; ++t) {
    if (!encode(&A->in[0][t], ins[t], dt, p.W, p.H, in_planes[t], pl.bw, pl.K, false)) return false;
    if (!encode(&A->in[1][t], ins[t], dt, p.W, p.H, in_planes[t], pl.K, pl.bh, true)) return false;
  }
  for (int t = 0; t < nout; ++t)
    if (!encode(&A->out[1][t], outs[t], dt, p.W, p.H, out_planes, pl.K, pl.cl > 1 ? pl.bhs : pl.bh, true))
      return false;
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
  if (const char* ev = knob("GSPN_GRID")) {  // experiments only: cap the persistent grid
    const int64_t g = atoll(ev);
    if (g > 0 && g < grid) grid = g;
  }
  if (A.plan.cl > 1) {  // P-split: clusters of cl CTAs, one chain per cluster at a time
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = A.plan.cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = A.plan.smem_bytes;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(static_cast<unsigned>(A.plan.cl * sm_count()), 1, 1);
    int ncl = 0;
    e = cudaOccupancyMaxActiveClusters(&ncl, kernel, &cfg);
    if (e != cudaSuccess) return e;
    if (ncl < 1) return cudaErrorInvalidConfiguration;
    if (ncl > A.plan.nchains) ncl = static_cast<int>(A.plan.nchains);
    cfg.gridDim = dim3(static_cast<unsigned>(ncl * A.plan.cl), 1, 1);
    e = cudaLaunchKernelEx(&cfg, kernel, A);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  if (grid > A.plan.nchains) grid = A.plan.nchains;
  kernel<<<static_cast<unsigned>(grid), threads, A.plan.smem_bytes, s>>>(A);
  return cudaGetLastError();
}

// GSPN-local chains (kchunk > 0) run the kLocal instantiations, with the pre-normalised or the clamped
// normaliser only (fewer instantiations; the clamped reciprocal is exact wherever S > 0).
template <typename T, bool kCl, bool kXG = false>
cudaError_t launch_fwd(int mode, bool local, const StreamArgs& A, cudaStream_t s) {
  if (local) {
    if (mode == kNormPre) return launch(fwd_stream_kernel<T, kNormPre, kCl, true, kXG>, A, s);
    return launch(fwd_stream_kernel<T, kNormClamp, kCl, true, kXG>, A, s);
  }
  if (mode == kNormPre) return launch(fwd_stream_kernel<T, kNormPre, kCl, false, kXG>, A, s);
  if (mode == kNormClamp) return launch(fwd_stream_kernel<T, kNormClamp, kCl, false, kXG>, A, s);
  return launch(fwd_stream_kernel<T, kNormFull, kCl, false, kXG>, A, s);
}
template <typename T, bool kCl>
cudaError_t launch_bwd(int mode, bool local, const StreamArgs& A, cudaStream_t s) {
  if (local) {
    if (mode == kNormPre) return launch(bwd_stream_kernel<T, kNormPre, kCl, true>, A, s);
    return launch(bwd_stream_kernel<T, kNormClamp, kCl, true>, A, s);
  }
  if (mode == kNormPre) return launch(bwd_stream_kernel<T, kNormPre, kCl, false>, A, s);
  if (mode == kNormClamp) return launch(bwd_stream_kernel<T, kNormClamp, kCl, false>, A, s);
  return launch(bwd_stream_kernel<T, kNormFull, kCl, false>, A, s);
}

int norm_mode(const ScanParams& p, const Plan& pl) {
  if (p.flags & GSPN_FLAG_PRENORMALIZED) return kNormPre;
  return (p.H % pl.K == 0 && p.W % pl.K == 0) ? kNormFull : kNormClamp;
}

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// Backward workspace: the adjoint state g [D, B, C, H, W] in the I/O dtype, then one readiness counter per
// (b, c) plane (single-launch backward).
struct WsLayout {
  size_t g, ready, total;
};

WsLayout ws_layout(int64_t B, int64_t C, int64_t H, int64_t W, int64_t D, gspn_dtype_t dt) {
  WsLayout l;
  l.g = 0;
  l.ready = align_up(static_cast<size_t>(D * B * C * H * W) * (dt == GSPN_BF16 ? 2 : 4));
  l.total = l.ready + align_up(static_cast<size_t>(B * C) * sizeof(unsigned));
  return l;
}

}  // namespace

size_t stream_bwd_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W, int64_t D, int64_t, gspn_dtype_t dt) {
  return ws_layout(B, C, H, W, D, dt).total;
}

cudaError_t launch_fwd_stream(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches, bool* handled,
                              const char** path) {
  *handled = false;
  // per call, on the heap (~2 KB): no shared launch state; the launch copies it into the parameter buffer
  std::unique_ptr<StreamArgs> hold(new StreamArgs());
  StreamArgs& A = *hold;
  memset(&A, 0, sizeof A);
  A.p = p;
  // Experiments only (GSPN_FWD_XG): x from global memory / L2 instead of the TMA ring (4 tiles per stage,
  // one more stage). Measured much slower on config 4 (fwd 4.72 vs 2.93 ms, profiles/r2_notes.md item 7).
  const int K = 32 / (dt == GSPN_BF16 ? 2 : 4);
  Plan probe;
  if (!make_plan(p, dt, F_NIN, &probe)) return cudaSuccess;
  const bool xg = probe.cl == 1 && p.W % K == 0 && knob("GSPN_FWD_XG");
  const int nin = xg ? F_NIN - 1 : F_NIN;
  if (!make_plan(p, dt, nin, &A.plan)) return cudaSuccess;
  if (p.ckpt != nullptr && (A.plan.cl > 1 || A.plan.npack > 1)) return cudaSuccess;  // checkpoints: see ckpt_eligible
  A.plan.no_h = p.hout == nullptr ? 1 : 0;
  if (!xg && A.plan.cl == 1 && A.plan.npack == 1 && p.W % K == 0 && knob("GSPN_HCP")) {
    A.plan.hcp = 1;
    A.plan.tx_hc = static_cast<uint32_t>((nin - 3) * A.plan.nbh * A.plan.bh * 32);
  }
  const void* ins_all[F_NIN] = {p.x, p.lam, p.wl, p.wm, p.wr};
  const int64_t planes_all[F_NIN] = {p.B * p.C, p.D * p.B * p.C, p.D * p.B * p.G, p.D * p.B * p.G, p.D * p.B * p.G};
  void* outs[1] = {p.hout};
  if (!fill_maps(&A, ins_all + (xg ? 1 : 0), nin, outs, planes_all + (xg ? 1 : 0), p.D * p.B * p.C,
                 p.hout != nullptr ? 1 : 0, dt))
    return cudaSuccess;
  *handled = true;
  using BF = __nv_bfloat16;
  const int mode = norm_mode(p, A.plan);
  cudaError_t e;
  const bool cl = A.plan.cl > 1;
  *path = cl ? "stream-cluster" : "stream";
  const bool local = p.kchunk > 0;
  if (dt == GSPN_BF16)
    e = cl ? launch_fwd<BF, true>(mode, local, A, s)
           : (xg ? launch_fwd<BF, false, true>(mode, local, A, s) : launch_fwd<BF, false>(mode, local, A, s));
  else
    e = cl ? launch_fwd<float, true>(mode, local, A, s)
           : (xg ? launch_fwd<float, false, true>(mode, local, A, s) : launch_fwd<float, false>(mode, local, A, s));
  *launches += 1;
  return e;
}

// Plan + tensor maps of the TMA-staged output kernel for `ncons` consumer warps within `budget` bytes of
// shared memory. Returns false if the shape does not fit.
bool setup_out_tma(const ScanParams& p, const void* g, gspn_dtype_t dt, bool vert_done, int ncons, int budget,
                   OutArgs& A, bool merged = false, bool all_done = false, bool allow_wide = false) {
  const bool grouped = p.G != p.C;
  memset(&A, 0, sizeof A);
  A.p = p;
  const int es = dt == GSPN_BF16 ? 2 : 4;
  // only where the caller launches a kWide instantiation
  A.wide = (allow_wide && p.W > 256 && p.W % 256 == 0 && p.W / 256 <= 256 && !knob("GSPN_OUT_NARROW")) ? 1 : 0;
  A.BX = A.wide ? static_cast<int>(p.W) : static_cast<int>(std::min<int64_t>(p.W, 256));
  A.nbx = static_cast<int>((p.W + A.BX - 1) / A.BX);
  const int D = static_cast<int>(p.D);
  auto pad = [](int64_t v) { return (v + 127) / 128 * 128; };
  const int nrb_t = grouped ? 2 : 5;  // RB-row tiles per direction: g, lam (+ w_l, w_m, w_r)
  auto stage_of = [&](int rb) {
    return A.nbx * (pad(es * A.BX * rb) * (1 + nrb_t * D) + pad(es * A.BX * (rb + 2)) * D);
  };
  // enough rows per unit to give every consumer thread a 4-column chunk, 2+ stages
  int RB = 1;
  // up to 32 rows per unit: short rows (config 2's 56 columns) need them to give every consumer a chunk
  // (16 -> 32: config 2 bwd 0.575 -> 0.480 ms); then equal row blocks, no mostly-empty last block
  int rbmax = 32;
  if (const char* e = knob("GSPN_OUT_RBMAX")) rbmax = std::max(1, std::min(64, atoi(e)));  // experiments
  while (RB < rbmax && RB * (p.W / 4) < ncons * 32) RB <<= 1;
  if (grouped) {  // exactly one chunk per thread: the group sums live in its registers
    while (RB > 1 && RB * (p.W / 4) > ncons * 32) RB >>= 1;
    if (p.W / 4 > ncons * 32) return false;
  }
  if (const char* e = knob("GSPN_OUT_RB"); e && !grouped) RB = std::max(1, std::min(128, atoi(e)));  // experiments
  while (RB > 1 && 2 * stage_of(RB) > budget) RB >>= 1;
  if (2 * stage_of(RB) > budget) return false;
  if (!grouped && !knob("GSPN_OUT_NOBAL")) {
    const int64_t nb = (p.H + RB - 1) / RB;
    RB = static_cast<int>((p.H + nb - 1) / nb);
  }
  A.RB = RB;
  A.box_rb = static_cast<uint32_t>(pad(es * A.BX * RB));
  A.box_h = static_cast<uint32_t>(pad(es * A.BX * (RB + 2)));
  A.tile_rb = A.nbx * A.box_rb;
  A.tile_h = A.nbx * A.box_h;
  A.per_k = nrb_t * A.tile_rb + A.tile_h;
  A.stage_bytes = A.tile_rb + D * A.per_k;
  {  // x (| dy) | direction k's tiles; a vertical direction of the hybrid backward holds only g and lam (and,
     // merged, the h halo tile for du)
    uint32_t o = A.tile_rb;
    A.dyoff = o;
    if (merged) o += A.tile_rb;
    for (int k = 0; k < D; ++k) {
      A.koff[k] = o;
      const bool vd = all_done || (vert_done && (p.dirbit[k] == GSPN_DIR_T2B || p.dirbit[k] == GSPN_DIR_B2T));
      A.khoff[k] = o + (vd ? 2 : nrb_t) * A.tile_rb;
      o += vd ? 2 * A.tile_rb + (merged ? A.tile_h : 0) : A.per_k;
    }
    A.stage_bytes = o;
  }
  A.tx = static_cast<uint32_t>(A.nbx * (es * A.BX * RB * (1 + nrb_t * D) + es * A.BX * (RB + 2) * D));  // payload
  if (vert_done) {  // vertical directions load g and lam only (+ the h halo when merged)
    int nv = 0;
    for (int k = 0; k < D; ++k) nv += (all_done || p.dirbit[k] == GSPN_DIR_T2B || p.dirbit[k] == GSPN_DIR_B2T) ? 1 : 0;
    A.tx -= static_cast<uint32_t>(A.nbx * nv * (es * A.BX * RB * (nrb_t - 2) + (merged ? 0 : es * A.BX * (RB + 2))));
  }
  if (merged) A.tx += static_cast<uint32_t>(A.nbx * es * A.BX * RB);  // dy
  A.nstages = static_cast<int>(std::min<int64_t>(6, budget / A.stage_bytes));
  A.nrb = static_cast<int>((p.H + RB - 1) / RB);
  A.nunits = (grouped ? p.B * p.G : p.B * p.C) * A.nrb;
  if (A.nunits >= (int64_t{1} << 31)) return false;  // 32-bit unit decode in the kernels
  const int64_t nc = p.D * p.B * p.C;
  const bool wd = A.wide != 0;
  bool ok = encode_rows(&A.x, p.x, dt, p.W, p.H, p.B * p.C, A.BX, RB, wd) &&
            encode_rows(&A.g, g, dt, p.W, p.H, nc, A.BX, RB, wd) &&
            encode_rows(&A.lam, p.lam, dt, p.W, p.H, nc, A.BX, RB, wd) &&
            encode_rows(&A.wl, p.wl, dt, p.W, p.H, nc, A.BX, RB, wd) &&
            encode_rows(&A.wm, p.wm, dt, p.W, p.H, nc, A.BX, RB, wd) &&
            encode_rows(&A.wr, p.wr, dt, p.W, p.H, nc, A.BX, RB, wd) &&
            encode_rows(&A.h, p.h, dt, p.W, p.H, nc, A.BX, RB + 2, wd);
  if (ok && merged) ok = encode_rows(&A.dy, p.dy, dt, p.W, p.H, p.B * p.C, A.BX, RB, wd);
  return ok;
}

uint32_t out_tma_smem(const OutArgs& A) { return 1024 + A.nstages * A.stage_bytes + 2 * 8 * A.nstages; }

// Forward + merge in one cooperative launch (gspn_fwd_merged). *handled = false when the shape takes
// another path (P-split chains, or B C H W not a multiple of the vector width): the caller falls back.
cudaError_t launch_fwd_merged(const ScanParams& p, gspn_dtype_t dt, const void* u, void* y, float scale,
                              cudaStream_t s, int* launches, bool* handled) {
  *handled = false;
  const int V = dt == GSPN_BF16 ? 8 : 4;
  const int64_t N = p.B * p.C * p.H * p.W;
  if (N % V != 0) return cudaSuccess;
  std::unique_ptr<OneFwdArgs> hold(new OneFwdArgs());
  OneFwdArgs& A = *hold;
  memset(&A, 0, sizeof A);
  A.s.p = p;
  if (!make_plan(p, dt, F_NIN, &A.s.plan) || A.s.plan.cl > 1) return cudaSuccess;
  const void* ins[F_NIN] = {p.x, p.lam, p.wl, p.wm, p.wr};
  const int64_t in_planes[F_NIN] = {p.B * p.C, p.D * p.B * p.C, p.D * p.B * p.G, p.D * p.B * p.G, p.D * p.B * p.G};
  void* outs[1] = {p.hout};
  if (!fill_maps(&A.s, ins, F_NIN, outs, in_planes, p.D * p.B * p.C, 1, dt)) return cudaSuccess;
  A.u = u;
  A.y = y;
  A.scale = scale;
  A.N = N;
  *handled = true;
  const int mode = norm_mode(p, A.s.plan);
  const bool local = p.kchunk > 0;
  auto go = [&](auto kernel) -> cudaError_t {
    const uint32_t smem = A.s.plan.smem_bytes;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int threads = (A.s.plan.nwc + 2) * 32;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int64_t grid = static_cast<int64_t>(sm_count()) * per_sm;  // every CTA resident (grid barrier)
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3(static_cast<unsigned>(grid), 1, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kernel, A);
    return e != cudaSuccess ? e : cudaGetLastError();
  };
  using BF = __nv_bfloat16;
  cudaError_t e;
  if (dt == GSPN_BF16) {
    if (local) e = mode == kNormPre ? go(fwd_one_kernel<BF, kNormPre, true>) : go(fwd_one_kernel<BF, kNormClamp, true>);
    else e = mode == kNormPre ? go(fwd_one_kernel<BF, kNormPre, false>)
             : mode == kNormClamp ? go(fwd_one_kernel<BF, kNormClamp, false>) : go(fwd_one_kernel<BF, kNormFull, false>);
  } else {
    if (local) e = mode == kNormPre ? go(fwd_one_kernel<float, kNormPre, true>) : go(fwd_one_kernel<float, kNormClamp, true>);
    else e = mode == kNormPre ? go(fwd_one_kernel<float, kNormPre, false>)
             : mode == kNormClamp ? go(fwd_one_kernel<float, kNormClamp, false>) : go(fwd_one_kernel<float, kNormFull, false>);
  }
  *launches += 1;
  return e;
}

// NEXT-3 eligibility (forward checkpoints and the recompute backward must agree): per-channel weights,
// unpacked, unsplit chains, H and W multiples of K, global scan, the backward plan (6 tiles) fits.
bool ckpt_eligible(const ScanParams& p, gspn_dtype_t dt) {
  if (p.G != p.C || p.kchunk > 0) return false;
  const int K = 32 / (dt == GSPN_BF16 ? 2 : 4);
  if (p.H % K != 0 || p.W % K != 0) return false;
  Plan pl;
  if (!make_plan(p, dt, R_NIN, &pl)) return false;
  return pl.cl == 1 && pl.npack == 1;
}

size_t ckpt_floats(const ScanParams& p, gspn_dtype_t dt) {
  const int KS = 16 / (dt == GSPN_BF16 ? 2 : 4);
  return static_cast<size_t>(p.D * p.B * p.C) * static_cast<size_t>(p.H * p.W / KS);
}

// TMA-staged output kernel. Returns false if the shape does not fit (caller falls back).
bool launch_out_tma(const ScanParams& p, const void* g, gspn_dtype_t dt, cudaStream_t s, cudaError_t* err,
                    bool vert_done = false, bool dry_run = false) {
  const bool grouped = p.G != p.C;
  if (knob("GSPN_OUT_REG")) return false;  // experiments: register-staged kernel
  std::unique_ptr<OutArgs> hold(new OutArgs());
  OutArgs& A = *hold;
  if (!setup_out_tma(p, g, dt, vert_done, kOutConsumers, smem_optin() - 1024 - 256, A, false, false, grouped)) return false;
  if (dry_run) return true;
  const uint32_t smem = out_tma_smem(A);
  using BF = __nv_bfloat16;
  auto kern = p.kchunk > 0
      ? (grouped ? (A.wide ? (dt == GSPN_BF16 ? bwd_out_grp_tma_kernel<BF, true, true> : bwd_out_grp_tma_kernel<float, true, true>)
                           : (dt == GSPN_BF16 ? bwd_out_grp_tma_kernel<BF, true> : bwd_out_grp_tma_kernel<float, true>))
                 : vert_done ? (dt == GSPN_BF16 ? bwd_out_tma_kernel<BF, true, true>
                                                : bwd_out_tma_kernel<float, true, true>)
                             : (dt == GSPN_BF16 ? bwd_out_tma_kernel<BF, true, false>
                                                : bwd_out_tma_kernel<float, true, false>))
      : (grouped ? (A.wide ? (dt == GSPN_BF16 ? bwd_out_grp_tma_kernel<BF, false, true> : bwd_out_grp_tma_kernel<float, false, true>)
                           : (dt == GSPN_BF16 ? bwd_out_grp_tma_kernel<BF, false> : bwd_out_grp_tma_kernel<float, false>))
                 : vert_done ? (dt == GSPN_BF16 ? bwd_out_tma_kernel<BF, false, true>
                                                : bwd_out_tma_kernel<float, false, true>)
                             : (dt == GSPN_BF16 ? bwd_out_tma_kernel<BF, false, false>
                                                : bwd_out_tma_kernel<float, false, false>));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e == cudaSuccess) {
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (kOutConsumers + 1) * 32, smem);
    if (e == cudaSuccess) {
      int64_t grid = static_cast<int64_t>(sm_count()) * std::max(per_sm, 1);
      if (grid > A.nunits) grid = A.nunits;
      kern<<<static_cast<unsigned>(grid), (kOutConsumers + 1) * 32, smem, s>>>(A);
      e = cudaGetLastError();
    }
  }
  *err = e;
  return true;
}

// Cooperative persistent launch of bwd_one_kernel: every CTA resident at once (the grid barrier needs
// it), grid = resident CTAs capped at the larger of the two phases' work-item counts.
template <typename KernelT>
cudaError_t launch_one(KernelT kernel, const OneArgs& A, cudaStream_t s) {
  const uint32_t smem = std::max<uint32_t>(A.s.plan.smem_bytes, out_tma_smem(A.o));
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int threads = (A.s.plan.nwc + 2) * 32;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = static_cast<int64_t>(sm_count()) * per_sm;
  grid = std::min<int64_t>(grid, std::max<int64_t>(A.s.plan.nchains, A.o.nunits));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.gridDim = dim3(static_cast<unsigned>(grid), 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kernel, A);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// dlam and dx of the fused backward (one elementwise launch over [B, C, H, W]).
template <typename T>
cudaError_t launch_dx(const ScanParams& p, const void* g, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  const int64_t N = p.B * p.C * p.H * p.W;
  const int64_t nv = N / V;
  int64_t blocks = (nv + 255) / 256;
  if (blocks > static_cast<int64_t>(sm_count()) * 8) blocks = static_cast<int64_t>(sm_count()) * 8;
  const T *x = static_cast<const T*>(p.x), *lam = static_cast<const T*>(p.lam), *gt = static_cast<const T*>(g);
  T *dl = static_cast<T*>(p.dlam), *dx = static_cast<T*>(p.dx);
  const unsigned b = static_cast<unsigned>(blocks < 1 ? 1 : blocks);
  switch (p.D) {
    case 1: bwd_dx_kernel<T, 1><<<b, 256, 0, s>>>(x, lam, gt, dl, dx, N, nv); break;
    case 2: bwd_dx_kernel<T, 2><<<b, 256, 0, s>>>(x, lam, gt, dl, dx, N, nv); break;
    case 3: bwd_dx_kernel<T, 3><<<b, 256, 0, s>>>(x, lam, gt, dl, dx, N, nv); break;
    default: bwd_dx_kernel<T, 4><<<b, 256, 0, s>>>(x, lam, gt, dl, dx, N, nv); break;
  }
  return cudaGetLastError();
}

// Recompute-h backward, one cooperative launch. Returns false (nothing launched) if not eligible.
bool launch_bwd_recompute(const ScanParams& p0, gspn_dtype_t dt, cudaStream_t s, int* launches, cudaError_t* err) {
  if (!ckpt_eligible(p0, dt)) return false;
  std::unique_ptr<OneArgs> one(new OneArgs());
  StreamArgs& A = one->s;
  memset(&A, 0, sizeof A);
  A.p = p0;
  ScanParams& p = A.p;
  if (!make_plan(p, dt, R_NIN, &A.plan)) return false;
  Plan& pl = A.plan;
  const WsLayout l = ws_layout(p.B, p.C, p.H, p.W, p.D, dt);
  if (p.ws == nullptr || p.ws_bytes < l.total || p.ckpt == nullptr) return false;
  A.g = static_cast<char*>(p.ws) + l.g;
  const int64_t nc = p.D * p.B * p.C;
  const void* ins[R_NIN] = {p.dh, p.wl, p.wm, p.wr, p.x, p.lam};
  const int64_t in_planes[R_NIN] = {nc, nc, nc, nc, p.B * p.C, nc};
  void* outs[4] = {A.g, p.dwl, p.dwm, p.dwr};
  if (!fill_maps(&A, ins, R_NIN, outs, in_planes, nc, 4, dt)) return false;
  if (!setup_out_tma(p, A.g, dt, true, pl.nwc, smem_optin() - 1024 - 256, one->o, false, true)) return false;
  const int mode = norm_mode(p, pl);
  using BF = __nv_bfloat16;
  cudaError_t e;
  if (dt == GSPN_BF16)
    e = mode == kNormPre ? launch_one(bwd_rc_kernel<BF, kNormPre>, *one, s)
        : mode == kNormClamp ? launch_one(bwd_rc_kernel<BF, kNormClamp>, *one, s)
                             : launch_one(bwd_rc_kernel<BF, kNormFull>, *one, s);
  else
    e = mode == kNormPre ? launch_one(bwd_rc_kernel<float, kNormPre>, *one, s)
        : mode == kNormClamp ? launch_one(bwd_rc_kernel<float, kNormClamp>, *one, s)
                             : launch_one(bwd_rc_kernel<float, kNormFull>, *one, s);
  *launches += 1;
  *err = e;
  return true;
}

// Fused backward for per-channel weights on unpacked, unsplit chains (the bench's config 4 shape):
// one persistent launch for the recurrence + tap gradients, one elementwise launch for dlam / dx.
// Returns false (nothing launched) when the shape takes the split path.
bool launch_bwd_fused(const ScanParams& p0, gspn_dtype_t dt, cudaStream_t s, int* launches, cudaError_t* err) {
  if (p0.G != p0.C || knob("GSPN_NOFUSE")) return false;
  std::unique_ptr<StreamArgs> hold(new StreamArgs());
  StreamArgs& A = *hold;
  const int es = dt == GSPN_BF16 ? 2 : 4;
  if ((p0.B * p0.C * p0.H * p0.W * es) % 16 != 0) return false;  // dx kernel: 16-byte vectors per slab
  memset(&A, 0, sizeof A);
  A.p = p0;
  ScanParams& p = A.p;
  // Horizontal chains' dw in the recurrence measured slower than the split (6.45 vs 3.98 ms bwd on
  // config 4's horizontal directions; profiles/r1_notes.md): by default only vertical chains are fused
  // and the output kernel forms the horizontal chains' dw (GSPN_FUSE_H=1: fuse both, experiments).
  const bool merged = p.dy != nullptr;  // gspn_bwd_merged: dh = s u dy on the fly, du written (single launch only)
  const bool fuse_h = !merged && knob("GSPN_FUSE_H") != nullptr;
  if (merged && (p.kchunk > 0 || knob("GSPN_TWO_LAUNCH"))) return false;
  // GSPN_HF (experiments): horizontal chains form their tap gradients in the recurrence too (kHF), from an
  // h tile with 48-byte rows (the tile's columns + one chunk towards step t-1); the output phase then forms
  // only dlam and dx. ~12% fewer algorithmic bytes, but measured slower than the hybrid (config 4 bwd
  // 6.90-6.94 vs 6.84-6.87 ms, config 2 0.64 vs 0.57 ms; profiles/r2_notes.md): the 6-slot stage leaves two
  // stages in flight and the storer's four tile stores hold each stage longer. Direct 16-byte stores from
  // registers instead of the in-place + TMA store: 11.5 ms (scattered partial-sector writes).
  // (kHF: the h tile has 48-byte rows = 1.5 slots; the stage holds 6 slots, merged would need 7: hybrid)
  bool hf = !fuse_h && !merged && p.kchunk == 0 && !knob("GSPN_TWO_LAUNCH") && knob("GSPN_HF");
  if (hf && (!make_plan(p, dt, B_NIN + 2, &A.plan) || A.plan.nstages < 2 || A.plan.cl > 1)) hf = false;
  if (!hf && !make_plan(p, dt, fuse_h ? B_NINF : B_NIN + 1 + (merged ? 1 : 0), &A.plan)) return false;
  Plan& pl = A.plan;
  const bool local = p.kchunk > 0;
  if (pl.cl > 1 || (fuse_h && (pl.npack > 1 || local)) || (knob("GSPN_NOFUSE_PACKED") && pl.npack > 1)) return false;
  pl.fuse_h = fuse_h ? 1 : 0;
  // make_plan counted pl.nin tiles per stage for both orientations: vertical loads B_NIN + 1 (no B_H1),
  // horizontal B_NIN (dh, w) unless fully fused; merged: + dy for both
  pl.tx_v = pl.tx_v / pl.nin * (B_NIN + 1 + (merged ? 1 : 0));
  if (!fuse_h) pl.tx_h = pl.tx_h / pl.nin * (B_NIN + (merged ? 1 : 0)) + (hf ? pl.tx_h / pl.nin / 2 * 3 : 0);
  const WsLayout l = ws_layout(p.B, p.C, p.H, p.W, p.D, dt);
  if (p.ws == nullptr || p.ws_bytes < l.total) return false;
  A.g = static_cast<char*>(p.ws) + l.g;
  const int64_t nc = p.D * p.B * p.C;
  const void* ins[B_NINF] = {p.dh, p.wl, p.wm, p.wr, p.h, merged ? p.dy : p.h};
  const int64_t in_planes[B_NINF] = {nc, nc, nc, nc, nc, merged ? p.B * p.C : nc};
  void* outs[4] = {A.g, p.dwl, p.dwm, p.dwr};
  if (!fill_maps(&A, ins, pl.nin, outs, in_planes, nc, (pl.fuse_h || hf) ? 4 : 1, dt)) return false;
  if (hf && !(pl.npack > 1 ? encode(&A.in[1][B_H0], p.h, dt, p.W, p.H, nc, pl.K + pl.K / 2, p.H, false, pl.npack)
                           : encode(&A.in[1][B_H0], p.h, dt, p.W, p.H, nc, pl.K + pl.K / 2, pl.bh, false)))
    return false;  // h with 48-byte rows (the tile's columns + one chunk towards step t-1)
  cudaError_t e0 = cudaSuccess;
  if (!pl.fuse_h && !launch_out_tma(p, A.g, dt, s, &e0, true, true)) return false;  // output kernel must fit
  const int mode = norm_mode(p, pl);
  if (!pl.fuse_h && !knob("GSPN_TWO_LAUNCH")) {  // single launch: recurrence | grid barrier | outputs
    std::unique_ptr<OneArgs> one(new OneArgs());
    one->s = A;
    const bool allow_wide = !merged && !hf && !local && dt == GSPN_BF16;  // the kWide instantiations
    if (setup_out_tma(p, A.g, dt, true, pl.nwc, smem_optin() - 1024 - 256, one->o, merged, hf, allow_wide)) {
      // Per-plane readiness instead of the grid-wide barrier (experiments only): measured slower, 7.03-7.08
      // vs 6.78-6.82 ms on config 4 (3 same-box pairs; profiles/r2_notes.md) -- early phase-2 units compete
      // with the last chains for bandwidth and every chain pays a gpu-scope fence.
      if (knob("GSPN_PLANE_READY")) {
        one->s.ready = reinterpret_cast<unsigned*>(static_cast<char*>(p.ws) + l.ready);
        one->o.ready = one->s.ready;
        one->o.npack = pl.npack;
      }
      cudaError_t e;
      using BF = __nv_bfloat16;
      if (hf) {
        if (dt == GSPN_BF16)
          e = mode == kNormPre ? launch_one(bwd_one_kernel<BF, kNormPre, false, false, true>, *one, s)
              : mode == kNormClamp ? launch_one(bwd_one_kernel<BF, kNormClamp, false, false, true>, *one, s)
                                   : launch_one(bwd_one_kernel<BF, kNormFull, false, false, true>, *one, s);
        else
          e = mode == kNormPre ? launch_one(bwd_one_kernel<float, kNormPre, false, false, true>, *one, s)
              : mode == kNormClamp ? launch_one(bwd_one_kernel<float, kNormClamp, false, false, true>, *one, s)
                                   : launch_one(bwd_one_kernel<float, kNormFull, false, false, true>, *one, s);
      } else if (merged) {
        if (dt == GSPN_BF16)
          e = mode == kNormPre ? launch_one(bwd_one_kernel<BF, kNormPre, false, true>, *one, s)
              : mode == kNormClamp ? launch_one(bwd_one_kernel<BF, kNormClamp, false, true>, *one, s)
                                   : launch_one(bwd_one_kernel<BF, kNormFull, false, true>, *one, s);
        else
          e = mode == kNormPre ? launch_one(bwd_one_kernel<float, kNormPre, false, true>, *one, s)
              : mode == kNormClamp ? launch_one(bwd_one_kernel<float, kNormClamp, false, true>, *one, s)
                                   : launch_one(bwd_one_kernel<float, kNormFull, false, true>, *one, s);
      } else if (dt == GSPN_BF16) {
        if (local) e = mode == kNormPre ? launch_one(bwd_one_kernel<BF, kNormPre, true>, *one, s)
                                        : launch_one(bwd_one_kernel<BF, kNormClamp, true>, *one, s);
        else if (one->o.wide)  // whole image rows per TMA box in the output phase (W > 256)
          e = mode == kNormPre ? launch_one(bwd_one_kernel<BF, kNormPre, false, false, false, true>, *one, s)
              : mode == kNormClamp ? launch_one(bwd_one_kernel<BF, kNormClamp, false, false, false, true>, *one, s)
                                   : launch_one(bwd_one_kernel<BF, kNormFull, false, false, false, true>, *one, s);
        else e = mode == kNormPre ? launch_one(bwd_one_kernel<BF, kNormPre, false>, *one, s)
                 : mode == kNormClamp ? launch_one(bwd_one_kernel<BF, kNormClamp, false>, *one, s)
                                      : launch_one(bwd_one_kernel<BF, kNormFull, false>, *one, s);
      } else {
        if (local) e = mode == kNormPre ? launch_one(bwd_one_kernel<float, kNormPre, true>, *one, s)
                                        : launch_one(bwd_one_kernel<float, kNormClamp, true>, *one, s);
        else e = mode == kNormPre ? launch_one(bwd_one_kernel<float, kNormPre, false>, *one, s)
                 : mode == kNormClamp ? launch_one(bwd_one_kernel<float, kNormClamp, false>, *one, s)
                                      : launch_one(bwd_one_kernel<float, kNormFull, false>, *one, s);
      }
      *launches += 1;
      *err = e;
      return true;
    }
  }
  if (merged) return false;  // the merged variant exists only as the single launch
  cudaError_t e;
  if (dt == GSPN_BF16) {
    using BF = __nv_bfloat16;
    if (local) e = mode == kNormPre ? launch(bwd_fused_kernel<BF, kNormPre, true>, A, s)
                                    : launch(bwd_fused_kernel<BF, kNormClamp, true>, A, s);
    else e = mode == kNormPre ? launch(bwd_fused_kernel<BF, kNormPre, false>, A, s)
             : mode == kNormClamp ? launch(bwd_fused_kernel<BF, kNormClamp, false>, A, s)
                                  : launch(bwd_fused_kernel<BF, kNormFull, false>, A, s);
  } else {
    if (local) e = mode == kNormPre ? launch(bwd_fused_kernel<float, kNormPre, true>, A, s)
                                    : launch(bwd_fused_kernel<float, kNormClamp, true>, A, s);
    else e = mode == kNormPre ? launch(bwd_fused_kernel<float, kNormPre, false>, A, s)
             : mode == kNormClamp ? launch(bwd_fused_kernel<float, kNormClamp, false>, A, s)
                                  : launch(bwd_fused_kernel<float, kNormFull, false>, A, s);
  }
  *launches += 1;
  if (e == cudaSuccess) {
    if (pl.fuse_h) {
      e = dt == GSPN_BF16 ? launch_dx<__nv_bfloat16>(p, A.g, s) : launch_dx<float>(p, A.g, s);
    } else if (!launch_out_tma(p, A.g, dt, s, &e, true)) {
      e = cudaErrorNotSupported;  // cannot happen for shapes make_plan accepted (checked below)
    }
    *launches += 1;
  }
  *err = e;
  return true;
}

cudaError_t launch_bwd_stream(const ScanParams& p0, gspn_dtype_t dt, cudaStream_t s, int* launches, bool* handled,
                              const char** path) {
  *handled = false;
  {
    cudaError_t e = cudaSuccess;
    if (launch_bwd_fused(p0, dt, s, launches, &e)) {
      *handled = true;
      *path = "stream-fused";
      return e;
    }
  }
  *path = "stream";
  if (p0.dy != nullptr) return cudaSuccess;  // merged backward: single-launch fused path only (caller falls back)
  std::unique_ptr<StreamArgs> hold(new StreamArgs());
  StreamArgs& A = *hold;
  memset(&A, 0, sizeof A);
  A.p = p0;
  ScanParams& p = A.p;
  if (!make_plan(p, dt, B_NIN, &A.plan)) return cudaSuccess;  // (W s) % 16 == 0: V-column groups tile W
  const WsLayout l = ws_layout(p.B, p.C, p.H, p.W, p.D, dt);
  if (p.ws == nullptr || p.ws_bytes < l.total) return cudaSuccess;
  A.g = static_cast<char*>(p.ws) + l.g;
  const void* ins[B_NIN] = {p.dh, p.wl, p.wm, p.wr};
  const int64_t nc = p.D * p.B * p.C, nw = p.D * p.B * p.G;
  const int64_t in_planes[B_NIN] = {nc, nw, nw, nw};
  void* outs[1] = {A.g};
  if (!fill_maps(&A, ins, B_NIN, outs, in_planes, nc, 1, dt)) return cudaSuccess;
  *handled = true;
  cudaError_t e;
  using BF = __nv_bfloat16;
  const int mode = norm_mode(p, A.plan);
  const bool cl = A.plan.cl > 1;
  if (cl) *path = "stream-cluster";
  const bool local = p.kchunk > 0;
  if (dt == GSPN_BF16) e = cl ? launch_bwd<BF, true>(mode, local, A, s) : launch_bwd<BF, false>(mode, local, A, s);
  else e = cl ? launch_bwd<float, true>(mode, local, A, s) : launch_bwd<float, false>(mode, local, A, s);
  *launches += 1;
  if (e != cudaSuccess) return e;
  const bool per_channel = p.G == p.C;
  if (launch_out_tma(p, A.g, dt, s, &e)) {
    *launches += 1;
    return e;
  }
  if (dt == GSPN_BF16)
    e = per_channel ? launch_out_pc<BF, 4>(p, A.g, s) : launch_out<BF, 4, false>(p, A.g, s);
  else
    e = per_channel ? launch_out_pc<float, 2>(p, A.g, s) : launch_out<float, 4, false>(p, A.g, s);
  *launches += 1;
  return e;
}

}  // namespace gspn
