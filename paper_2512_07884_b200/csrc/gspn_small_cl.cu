// gspn_small_cl.cu — grouped small planes (G < C, max(H, W) <= 32) on thread-block clusters: the
// compact-channel shapes of the paper (28 x 28 stages whose C channels share one affinity per group,
// PAPER.md:140-148 Eq. 3).
//
// Work decomposition: one CTA per (unit (b, g), direction k); the D direction CTAs of a
// unit form a cluster. A CTA normalises its direction's taps ONCE (a3: once per (d, b, g, t, r), shared by the
// group's C/G channels) and then streams the group's channels through two shared-memory batch buffers filled
// by 1D bulk copies (cp.async.bulk, one per plane -- rows of 28 x 2 bytes are too short for TMA tiles): the
// copies of batch i+2 land while batch i+1 is computed. Compute warps run one channel each (lane = position
// r, neighbours by warp shuffle, carry in fp32 registers, the next step's operands prefetched).
//
// Forward (a4/a5): h over lam in shared memory, written back by bulk stores (a producer warp issues every
// copy, so the compute warps never wait on a store).
// Backward (a6/a7): the adjoint recurrence leaves g_t (fp32) in the shared-memory rows it has consumed (bf16
// I/O: the high half over dh[t], the low half over h[t] -- h[t] was last read at step t+1); the tap gradients
// Da / Db / Dc of the direction are summed over ALL the group's channels in registers (one accumulator per
// step and lane), so dw is formed in-CTA through the normalisation Jacobian with no workspace and no atomics.
// dx = sum_d g_d lam_d needs the D directions: after each batch the CTAs signal each other through mbarriers
// (release / acquire at cluster scope; waited by spinning -- a suspend-time hint on a barrier completed by a
// remote arrive measured slower) and CTA k sums its share of the batch's pixels over the D CTAs' shared memory
// (distributed shared memory, fixed order). A unit of <= 8 channels runs as one batch with two chains per warp.
// Every reduction has a fixed order: bitwise deterministic.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "gspn_common.cuh"
#include "gspn_internal.h"
#include "gspn_ptx.cuh"

namespace gspn {
namespace {

using namespace ptx;

constexpr int kLMax = 32;     // small planes: L, P <= 32
constexpr int kFwdWarps = 4;  // forward compute warps (+ 1 producer warp)
constexpr int kFwdKc = 2;     // forward: channels per warp per batch (independent chains: ILP)
constexpr int kBwdWarps = 4;  // backward compute warps (one channel each per batch)

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint4 ld_cluster_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

// Normalised taps of direction k of unit (b, g) in scan order: TP[t P + r] = (a, b, c, 0) (
// DESIGN.md R1/R2), from the raw planes RAW[3][HW] (canonical pixel order) staged in shared memory.
template <typename T>
__device__ void taps_from_raw(const ScanParams& p, const DirGeom& gm, const T* RAW, int HW, float4* TP, int tid,
                              int nthr) {
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  const int P = static_cast<int>(gm.P);
  for (int idx = tid; idx < HW; idx += nthr) {
    const int t = idx / P, r = idx - t * P;
    const int pix = static_cast<int>(gm.base + t * gm.ts + r * gm.rs);
    const Taps tp = make_taps(to_f(RAW[pix]), to_f(RAW[HW + pix]), to_f(RAW[2 * HW + pix]), r >= 1, r <= P - 2, prenorm);
    TP[idx] = make_float4(tp.a, tp.b, tp.c, 0.f);
  }
}

// Shared-memory carve-up common to both kernels (byte offsets; every region 16-byte aligned).
struct ClLayout {
  uint32_t tp, raw, buf, bufb, part, bars, total;
};
__host__ __device__ __forceinline__ ClLayout cl_layout(int HW, int es, int kb, int nplanes, uint32_t min_part,
                                                      int nbuf = 2) {
  ClLayout L;
  const uint32_t pb = static_cast<uint32_t>(HW * es);
  L.tp = 0;
  L.raw = static_cast<uint32_t>(HW) * 16u;
  L.buf = L.raw + 3u * pb;
  L.bufb = static_cast<uint32_t>(kb * nplanes) * pb;
  L.part = L.buf + static_cast<uint32_t>(nbuf) * L.bufb;  // backward: per-warp fp32 tap-gradient partial sums
  L.bars = L.part + (min_part + 15u) / 16u * 16u;
  L.total = L.bars + 8 * 8;  // up to 7 mbarriers
  return L;
}

// ------------------------------------------------------------------------------------------ forward
// buffers: [2][kb][x | lam (-> h)]; warps [0, kFwdWarps) compute (kFwdKc channels each per batch), warp
// kFwdWarps produces (loads, and the stores of finished batches before their buffer is refilled).
template <typename T, bool kLocal>
__global__ void __launch_bounds__((kFwdWarps + 1) * 32) fwd_grp_cl_kernel(ScanParams p, int kb) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int H = static_cast<int>(p.H), W = static_cast<int>(p.W), HW = H * W, D = static_cast<int>(p.D);
  const int64_t Cg = p.C / p.G;
  const int k = static_cast<int>(blockIdx.x % D);
  const int64_t unit = blockIdx.x / D, b = unit / p.G, g = unit % p.G;
  const uint32_t pb = static_cast<uint32_t>(HW) * sizeof(T);
  const ClLayout Ly = cl_layout(HW, sizeof(T), kb, 2, 0);
  float4* TP = reinterpret_cast<float4*>(sm + Ly.tp);
  const T* RAW = reinterpret_cast<const T*>(sm + Ly.raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Ly.bars);  // [0] taps, [1, 2] full, [3, 4] done
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = static_cast<int>((Cg + kb - 1) / kb);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&bars[1 + s]), 1);
      mbar_init(smem_u32(&bars[3 + s]), kFwdWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t chain0 = (static_cast<int64_t>(k) * p.B + b) * p.C + g * Cg;  // lam / h plane of channel 0
  const int64_t xplane0 = b * p.C + g * Cg;
  auto nch = [&](int i) { return static_cast<int>(std::min<int64_t>(kb, Cg - static_cast<int64_t>(i) * kb)); };
  auto slot = [&](int s, int ch, int q) { return Ly.buf + (static_cast<uint32_t>(s) * kb * 2 + ch * 2 + q) * pb; };
  if (warp == kFwdWarps) {  // producer
    if (lane == 0) {
      const uint32_t tb = smem_u32(&bars[0]);
      mbar_arrive_tx(tb, 3 * pb);
      const int64_t wpl = ((static_cast<int64_t>(k) * p.B + b) * p.G + g) * HW;
      bulk_g2s(smem_u32(sm + Ly.raw), static_cast<const T*>(p.wl) + wpl, pb, tb);
      bulk_g2s(smem_u32(sm + Ly.raw + pb), static_cast<const T*>(p.wm) + wpl, pb, tb);
      bulk_g2s(smem_u32(sm + Ly.raw + 2 * pb), static_cast<const T*>(p.wr) + wpl, pb, tb);
      auto store = [&](int i) {
        const int s = i & 1;
        mbar_wait_sleep(smem_u32(&bars[3 + s]), (i >> 1) & 1);
        for (int c = 0; c < nch(i); ++c)
          bulk_s2g(static_cast<T*>(p.hout) + (chain0 + static_cast<int64_t>(i) * kb + c) * HW,
                   smem_u32(sm + slot(s, c, 1)), pb);
        bulk_commit();
      };
      for (int i = 0; i < nb; ++i) {
        const int s = i & 1;
        if (i >= 2) {  // batch i-2's h leaves the buffer before batch i's inputs land in it
          store(i - 2);
          bulk_wait_read0();
        }
        const uint32_t fb = smem_u32(&bars[1 + s]);
        mbar_arrive_tx(fb, 2 * pb * nch(i));
        for (int c = 0; c < nch(i); ++c) {
          const int64_t cc = static_cast<int64_t>(i) * kb + c;
          bulk_g2s(smem_u32(sm + slot(s, c, 0)), static_cast<const T*>(p.x) + (xplane0 + cc) * HW, pb, fb);
          bulk_g2s(smem_u32(sm + slot(s, c, 1)), static_cast<const T*>(p.lam) + (chain0 + cc) * HW, pb, fb);
        }
      }
      for (int i = std::max(nb - 2, 0); i < nb; ++i) store(i);
      bulk_wait_all();
    }
    return;
  }
  const uint32_t dir = p.dirbit[k];
  const DirGeom gm = dir_geom(dir, H, W);
  const int L = static_cast<int>(gm.L), P = static_cast<int>(gm.P);
  const int ts = static_cast<int>(gm.ts);
  mbar_wait_sleep(smem_u32(&bars[0]), 0);
  taps_from_raw<T>(p, gm, RAW, HW, TP, threadIdx.x, kFwdWarps * 32);
  named_bar(1, kFwdWarps * 32);
  const bool in = lane < P;
  const int r = in ? lane : 0;
  const int off0 = static_cast<int>(gm.base) + r * static_cast<int>(gm.rs);
  const int kcn = static_cast<int>(p.kchunk);
  for (int i = 0; i < nb; ++i) {
    const int s = i & 1;
    mbar_wait_sleep(smem_u32(&bars[1 + s]), (i >> 1) & 1);
    const int c0 = warp * kFwdKc;
    if (c0 < nch(i)) {
      const bool two = c0 + 1 < nch(i);
      const T* X0 = reinterpret_cast<const T*>(sm + slot(s, c0, 0));
      T* L0 = reinterpret_cast<T*>(sm + slot(s, c0, 1));
      const T* X1 = reinterpret_cast<const T*>(sm + slot(s, two ? c0 + 1 : c0, 0));
      T* L1 = reinterpret_cast<T*>(sm + slot(s, two ? c0 + 1 : c0, 1));
      // lanes >= P read only x (never written): no race with lane 0's in-place h stores
      const T* L0r = in ? L0 : X0;
      const T* L1r = in ? L1 : X1;
      float h0 = 0.f, h1 = 0.f;
      int off = off0;
      float x0 = to_f(X0[off]), l0 = to_f(L0r[off]), x1 = to_f(X1[off]), l1 = to_f(L1r[off]);
      float4 q = TP[r];
      for (int t = 0; t < L; ++t) {
        // operands of step t+1 (a different pixel from the one stored below)
        const int offn = t + 1 < L ? off + ts : off;
        const float nx0 = to_f(X0[offn]), nl0 = to_f(L0r[offn]), nx1 = to_f(X1[offn]), nl1 = to_f(L1r[offn]);
        const float4 nq = TP[(t + 1 < L ? t + 1 : t) * P + r];
        if constexpr (kLocal) {
          if (seg_start_step(dir, t, L, kcn)) h0 = h1 = 0.f;  // warp-uniform
        }
        const float u0 = __shfl_up_sync(0xffffffffu, h0, 1), d0 = __shfl_down_sync(0xffffffffu, h0, 1);
        const float u1 = __shfl_up_sync(0xffffffffu, h1, 1), d1 = __shfl_down_sync(0xffffffffu, h1, 1);
        const float v0 = fmaf(q.x, u0, fmaf(q.y, h0, fmaf(q.z, d0, l0 * x0)));
        const float v1 = fmaf(q.x, u1, fmaf(q.y, h1, fmaf(q.z, d1, l1 * x1)));
        if (in) {
          L0[off] = from_f<T>(v0);
          if (two) L1[off] = from_f<T>(v1);
        }
        h0 = in ? v0 : 0.f;
        h1 = in ? v1 : 0.f;
        off = offn;
        x0 = nx0; l0 = nl0; x1 = nx1; l1 = nl1; q = nq;
      }
    }
    fence_proxy_async();  // in-place h (generic proxy) -> visible to the producer's bulk stores
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&bars[3 + s]));
  }
}

// ------------------------------------------------------------------------------------------ backward
// buffers: [2][kb][x | lam | dh (-> g hi / dlam source) | h (-> g lo)]; all threads compute; thread 0 issues
// the bulk loads between the cluster barriers.
template <typename T>
__device__ __forceinline__ float g_at(const uint8_t* dhp, const uint8_t* hp, int px) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t hi = reinterpret_cast<const uint16_t*>(dhp)[px];
    const uint32_t lo = reinterpret_cast<const uint16_t*>(hp)[px];
    return __uint_as_float((hi << 16) | lo);
  } else {
    return reinterpret_cast<const float*>(dhp)[px];
  }
}
template <typename T>
__device__ __forceinline__ void g_put(uint8_t* dhp, uint8_t* hp, int px, float g) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t u = __float_as_uint(g);
    reinterpret_cast<uint16_t*>(dhp)[px] = static_cast<uint16_t>(u >> 16);
    reinterpret_cast<uint16_t*>(hp)[px] = static_cast<uint16_t>(u & 0xFFFFu);
  } else {
    reinterpret_cast<float*>(dhp)[px] = g;
  }
}
// V = 16 bytes of elements: g of V consecutive pixels from the (dh, h) 16-byte pieces.
template <typename T>
__device__ __forceinline__ void g_vec(const uint4& dh16, const uint4& h16, float (&g)[16 / sizeof(T)]) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t a[4] = {dh16.x, dh16.y, dh16.z, dh16.w}, c[4] = {h16.x, h16.y, h16.z, h16.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      g[2 * i] = __uint_as_float((a[i] << 16) | (c[i] & 0xFFFFu));
      g[2 * i + 1] = __uint_as_float((a[i] & 0xFFFF0000u) | (c[i] >> 16));
    }
  } else {
    g[0] = __uint_as_float(dh16.x); g[1] = __uint_as_float(dh16.y);
    g[2] = __uint_as_float(dh16.z); g[3] = __uint_as_float(dh16.w);
  }
}
template <typename T>
__device__ __forceinline__ void e_vec(const uint4& u, float (&v)[16 / sizeof(T)]) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t a[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(a[i] << 16);
      v[2 * i + 1] = __uint_as_float(a[i] & 0xFFFF0000u);
    }
  } else {
    v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y); v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
  }
}
template <typename T>
__device__ __forceinline__ uint4 pack_vec(const float (&v)[16 / sizeof(T)]) {
  if constexpr (sizeof(T) == 2) {
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      o[i] = *reinterpret_cast<uint32_t*>(&b2);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
  } else {
    return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3]));
  }
}

// kKc channels per compute warp per batch (2: a unit of <= 8 channels in ONE batch with a single buffer, the
// two chains interleaved step by step for ILP; 1: batches of kBwdWarps channels, double-buffered).
template <typename T, bool kLocal, int kKc>
__global__ void __launch_bounds__((kBwdWarps + 1) * 32, 2) bwd_grp_cl_kernel(ScanParams p, int kb) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int V = 16 / static_cast<int>(sizeof(T));
  const int H = static_cast<int>(p.H), W = static_cast<int>(p.W), HW = H * W, D = static_cast<int>(p.D);
  const int64_t Cg = p.C / p.G;
  const int k = static_cast<int>(cluster_ctarank());
  const int64_t unit = blockIdx.x / D, b = unit / p.G, g = unit % p.G;
  const uint32_t pb = static_cast<uint32_t>(HW) * sizeof(T);
  const ClLayout Ly = cl_layout(HW, sizeof(T), kb, 4, static_cast<uint32_t>(kBwdWarps * 3 * HW * 4), kKc == 2 ? 1 : 2);
  float4* TP = reinterpret_cast<float4*>(sm + Ly.tp);
  const T* RAW = reinterpret_cast<const T*>(sm + Ly.raw);
  // [0] taps, [1, 2] full (TMA bytes), [3, 4] ready (one arrive per cluster CTA: its g of the batch in the
  // slot is complete), [5, 6] free (one arrive per cluster CTA: done reading this CTA's slot)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Ly.bars);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  constexpr int NT = kBwdWarps * 32;
  const int nb = static_cast<int>((Cg + kb - 1) / kb);
  const int64_t chain0 = (static_cast<int64_t>(k) * p.B + b) * p.C + g * Cg;
  const int64_t xplane0 = b * p.C + g * Cg;
  auto nch = [&](int i) { return static_cast<int>(std::min<int64_t>(kb, Cg - static_cast<int64_t>(i) * kb)); };
  auto slot = [&](int s, int ch, int q) { return Ly.buf + (static_cast<uint32_t>(s) * kb * 4 + ch * 4 + q) * pb; };
  if (tid == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&bars[1 + s]), 1);
      mbar_init(smem_u32(&bars[3 + s]), D);
      mbar_init(smem_u32(&bars[5 + s]), D);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();  // every CTA's barriers initialised before any remote arrive
  if (warp == kBwdWarps) {  // producer: taps, then each batch once the cluster has released its slot
    if (lane == 0) {
      const uint32_t tb = smem_u32(&bars[0]);
      mbar_arrive_tx(tb, 3 * pb);
      const int64_t wpl = ((static_cast<int64_t>(k) * p.B + b) * p.G + g) * HW;
      bulk_g2s(smem_u32(sm + Ly.raw), static_cast<const T*>(p.wl) + wpl, pb, tb);
      bulk_g2s(smem_u32(sm + Ly.raw + pb), static_cast<const T*>(p.wm) + wpl, pb, tb);
      bulk_g2s(smem_u32(sm + Ly.raw + 2 * pb), static_cast<const T*>(p.wr) + wpl, pb, tb);
      for (int i = 0; i < nb; ++i) {
        const int s = i & 1;
        if (i >= 2) mbar_wait_cluster(smem_u32(&bars[5 + s]), ((i - 2) >> 1) & 1);
        const uint32_t fb = smem_u32(&bars[1 + s]);
        mbar_arrive_tx(fb, 4 * pb * nch(i));
        for (int c = 0; c < nch(i); ++c) {
          const int64_t cc = static_cast<int64_t>(i) * kb + c;
          bulk_g2s(smem_u32(sm + slot(s, c, 0)), static_cast<const T*>(p.x) + (xplane0 + cc) * HW, pb, fb);
          bulk_g2s(smem_u32(sm + slot(s, c, 1)), static_cast<const T*>(p.lam) + (chain0 + cc) * HW, pb, fb);
          bulk_g2s(smem_u32(sm + slot(s, c, 2)), static_cast<const T*>(p.dh) + (chain0 + cc) * HW, pb, fb);
          bulk_g2s(smem_u32(sm + slot(s, c, 3)), static_cast<const T*>(p.h) + (chain0 + cc) * HW, pb, fb);
        }
      }
    }
    __syncwarp();
    cluster_sync_all();  // matches the compute warps' final cluster barrier
    return;
  }
  const uint32_t dir = p.dirbit[k];
  const DirGeom gm = dir_geom(dir, H, W);
  const int L = static_cast<int>(gm.L), P = static_cast<int>(gm.P);
  const int ts = static_cast<int>(gm.ts), rs = static_cast<int>(gm.rs);
  mbar_wait_sleep(smem_u32(&bars[0]), 0);
  taps_from_raw<T>(p, gm, RAW, HW, TP, tid, NT);
  named_bar(1, NT);
  const bool in = lane < P;
  const int r = in ? lane : 0;
  const bool hl = in && r >= 1, hr = in && r <= P - 2;
  const int offr = static_cast<int>(gm.base) + r * rs;
  const int kcn = static_cast<int>(p.kchunk);
  // tap-gradient group sums of this lane's position, per step (reverse order index s = L-1-t)
  float* part = reinterpret_cast<float*>(sm + Ly.part);  // [warp][3][HW] in scan order (t P + r)
  for (int q = tid; q < kBwdWarps * 3 * HW; q += NT) part[q] = 0.f;
  for (int i = 0; i < nb; ++i) {
    const int sb = i & 1;
    const uint32_t par = (i >> 1) & 1;
    mbar_wait_sleep(smem_u32(&bars[1 + sb]), par);
    if (warp * kKc < nch(i)) {
      const T* DHr[kKc];
      const T* HSr[kKc];
      uint8_t* DHw[kKc];
      uint8_t* HSw[kKc];
      bool act[kKc];
      float ea[kKc], eb[kKc], ec[kKc], dhv[kKc], hv[kKc];
      int off = offr + (L - 1) * ts;
#pragma unroll
      for (int j = 0; j < kKc; ++j) {
        act[j] = warp * kKc + j < nch(i);
        const int c = act[j] ? warp * kKc + j : warp * kKc;
        const T* X = reinterpret_cast<const T*>(sm + slot(sb, c, 0));
        // lanes >= P read only x (never written)
        DHr[j] = in ? reinterpret_cast<const T*>(sm + slot(sb, c, 2)) : X;
        HSr[j] = in ? reinterpret_cast<const T*>(sm + slot(sb, c, 3)) : X;
        DHw[j] = sm + slot(sb, c, 2);
        HSw[j] = sm + slot(sb, c, 3);
        ea[j] = eb[j] = ec[j] = 0.f;
        dhv[j] = to_f(DHr[j][off]);
        hv[j] = L >= 2 ? to_f(HSr[j][off - ts]) : 0.f;
      }
      // the warp's tap-gradient partial sums at (t, r), scan order: this lane owns these words
      float* pa = part + (warp * 3 + 0) * HW + (L - 1) * P + r;
#pragma unroll 4
      for (int s = 0; s < L; ++s) {
        const int t = L - 1 - s;
        const float4 q = TP[t * P + r];
        bool seg = t == 0;
        if constexpr (kLocal) seg = seg_start_step(dir, t, L, kcn);
        float sa = 0.f, sbb = 0.f, sc = 0.f;
#pragma unroll
        for (int j = 0; j < kKc; ++j) {
          // operands of step t-1 (pixels of rows t-1 / t-2: not written at this step)
          const float ndh = t >= 1 ? to_f(DHr[j][off - ts]) : 0.f;
          const float nh = t >= 2 ? to_f(HSr[j][off - 2 * ts]) : 0.f;
          const float from_r = __shfl_down_sync(0xffffffffu, ea[j], 1);  // a_{t+1}[r+1] g_{t+1}[r+1]
          const float from_l = __shfl_up_sync(0xffffffffu, ec[j], 1);    // c_{t+1}[r-1] g_{t+1}[r-1]
          const float gt = in ? dhv[j] + eb[j] + ((hr ? from_r : 0.f) + (hl ? from_l : 0.f)) : 0.f;
          const float hc = (seg || !in) ? 0.f : hv[j];  // h_{t-1}[r] (0 at a segment start)
          const float hlv = __shfl_up_sync(0xffffffffu, hc, 1), hrv = __shfl_down_sync(0xffffffffu, hc, 1);
          if (act[j]) {
            sa = fmaf(gt, hl ? hlv : 0.f, sa);
            sbb = fmaf(gt, hc, sbb);
            sc = fmaf(gt, hr ? hrv : 0.f, sc);
          }
          ea[j] = q.x * gt;
          eb[j] = q.y * gt;
          ec[j] = q.z * gt;
          if constexpr (kLocal) {
            if (seg) ea[j] = eb[j] = ec[j] = 0.f;  // h_t did not depend on h_{t-1}
          }
          if (in && act[j]) g_put<T>(DHw[j], HSw[j], off, gt);  // over dh[t] (read) and h[t] (last read at t+1)
          dhv[j] = ndh;
          hv[j] = nh;
        }
        if (in) {
          pa[0] += sa;
          pa[HW] += sbb;
          pa[2 * HW] += sc;
        }
        pa -= P;
        off -= ts;
      }
    }
    // publish this CTA's g of batch i to the cluster (release), then wait for every direction's (acquire)
    named_bar(1, NT);
    if (tid == 0)
      for (int j = 0; j < D; ++j) mbar_arrive_remote(mapa(smem_u32(&bars[3 + sb]), static_cast<uint32_t>(j)));
    mbar_wait_cluster(smem_u32(&bars[3 + sb]), par);
    {
      const int nvp = HW / V;  // 16-byte vectors per plane
      const int nv = nch(i) * nvp;
      // dlam_k = g_k x (own CTA)
      for (int v = tid; v < nv; v += NT) {
        const int c = v / nvp, e0 = (v - c * nvp) * V;
        float gg[V], xx[V], o[V];
        g_vec<T>(*reinterpret_cast<const uint4*>(sm + slot(sb, c, 2) + e0 * sizeof(T)),
                 *reinterpret_cast<const uint4*>(sm + slot(sb, c, 3) + e0 * sizeof(T)), gg);
        e_vec<T>(*reinterpret_cast<const uint4*>(sm + slot(sb, c, 0) + e0 * sizeof(T)), xx);
#pragma unroll
        for (int e = 0; e < V; ++e) o[e] = gg[e] * xx[e];
        *reinterpret_cast<uint4*>(static_cast<T*>(p.dlam) + (chain0 + static_cast<int64_t>(i) * kb + c) * HW + e0) =
            pack_vec<T>(o);
      }
      // dx = sum_d g_d lam_d over the cluster's D CTAs (fixed order); CTA k takes vectors k, k + D, ...
      for (int v = k + D * tid; v < nv; v += D * NT) {
        const int c = v / nvp, e0 = (v - c * nvp) * V;
        const uint32_t a_dh = smem_u32(sm + slot(sb, c, 2) + e0 * sizeof(T));
        const uint32_t a_h = smem_u32(sm + slot(sb, c, 3) + e0 * sizeof(T));
        const uint32_t a_l = smem_u32(sm + slot(sb, c, 1) + e0 * sizeof(T));
        uint4 rdh[4], rh[4], rl[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // every remote load in flight before the first use
          if (j < D) {
            const uint32_t rj = static_cast<uint32_t>(j);
            rdh[j] = ld_cluster_v4(mapa(a_dh, rj));
            rh[j] = sizeof(T) == 2 ? ld_cluster_v4(mapa(a_h, rj)) : rdh[j];
            rl[j] = ld_cluster_v4(mapa(a_l, rj));
          }
        }
        float acc[V];
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j < D) {
            float gg[V], ll[V];
            g_vec<T>(rdh[j], rh[j], gg);
            e_vec<T>(rl[j], ll);
#pragma unroll
            for (int e = 0; e < V; ++e) acc[e] = fmaf(gg[e], ll[e], acc[e]);
          }
        }
        *reinterpret_cast<uint4*>(static_cast<T*>(p.dx) + (xplane0 + static_cast<int64_t>(i) * kb + c) * HW + e0) =
            pack_vec<T>(acc);
      }
    }
    // done reading every CTA's slot sb: release it (the producers refill it with batch i + 2)
    fence_proxy_async();
    named_bar(1, NT);
    if (tid == 0)
      for (int j = 0; j < D; ++j) mbar_arrive_remote(mapa(smem_u32(&bars[5 + sb]), static_cast<uint32_t>(j)));
  }
  // the peers' last reads of this CTA's slots are complete before this CTA may exit
  for (int i = std::max(nb - 2, 0); i < nb; ++i) mbar_wait_cluster(smem_u32(&bars[5 + (i & 1)]), (i >> 1) & 1);
  // dw: the warps' partial sums added in warp order, then the normalisation Jacobian (a7)
  named_bar(1, NT);
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  const bool f32out = p.flags & GSPN_FLAG_DW_F32;
  const int nw = static_cast<int>(std::min<int64_t>(kBwdWarps, Cg));
  const int64_t wpl = ((static_cast<int64_t>(k) * p.B + b) * p.G + g) * HW;
  for (int q = tid; q < HW; q += NT) {
    const int t = q / P, rr = q - t * P;
    const int pix = static_cast<int>(gm.base + t * gm.ts + rr * gm.rs);
    float Da = 0.f, Db = 0.f, Dc = 0.f;
    for (int w = 0; w < nw; ++w) {
      Da += part[(w * 3 + 0) * HW + q];
      Db += part[(w * 3 + 1) * HW + q];
      Dc += part[(w * 3 + 2) * HW + q];
    }
    float ol, om, orr;
    jacobian(to_f(RAW[pix]), to_f(RAW[HW + pix]), to_f(RAW[2 * HW + pix]), rr >= 1, rr <= P - 2, prenorm, Da, Db, Dc,
             ol, om, orr);
    if (f32out) {
      static_cast<float*>(p.dwl)[wpl + pix] = ol;
      static_cast<float*>(p.dwm)[wpl + pix] = om;
      static_cast<float*>(p.dwr)[wpl + pix] = orr;
    } else {
      static_cast<T*>(p.dwl)[wpl + pix] = from_f<T>(ol);
      static_cast<T*>(p.dwm)[wpl + pix] = from_f<T>(om);
      static_cast<T*>(p.dwr)[wpl + pix] = from_f<T>(orr);
    }
  }
  __syncwarp();
  cluster_sync_all();  // no CTA leaves while a peer may still arrive on its barriers
}

// channels per batch within the shared-memory budget (2+ CTAs per SM when possible)
int cl_batch(const ScanParams& p, int es, bool bwd, int kc = 1) {
  const int HW = static_cast<int>(p.H * p.W);
  const int64_t Cg = p.C / p.G;
  const uint32_t budget = static_cast<uint32_t>(device_smem_optin());
  const int maxkb = bwd ? kBwdWarps * kc : kFwdWarps * kFwdKc;
  const uint32_t minb2 = bwd ? static_cast<uint32_t>(kBwdWarps * 3 * HW * 4) : 0u;
  const int nbuf = bwd && kc == 2 ? 1 : 2;
  int kb = static_cast<int>(std::min<int64_t>(maxkb, Cg));
  while (kb > 1 && cl_layout(HW, es, kb, bwd ? 4 : 2, minb2, nbuf).total > budget) --kb;
  return cl_layout(HW, es, kb, bwd ? 4 : 2, minb2, nbuf).total <= budget ? kb : 0;
}

bool knob_set_cl(const char* name) {  // experiment knob (A/B tooling): read only when GSPN_EXPERIMENTS is set
  static const bool on = getenv("GSPN_EXPERIMENTS") != nullptr;
  return on && getenv(name) != nullptr;
}

template <typename K>
cudaError_t launch_cl(K kern, const ScanParams& p, int threads, int kb, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(p.D);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(static_cast<unsigned>(p.B * p.G * p.D), 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, p, kb);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

// Eligible: grouped weights on small planes whose planes are whole 16-byte vectors at 16-byte aligned bases
// (one bulk copy per plane), L, P <= 32, grid within limits.
bool small_cl_eligible(const ScanParams& p, gspn_dtype_t dt, bool bwd) {
  const int es = dt == GSPN_BF16 ? 2 : 4;
  if (p.G >= p.C || p.H > kLMax || p.W > kLMax || p.D < 1 || p.D > 4) return false;
  if ((p.H * p.W * es) % 16 != 0) return false;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p.x) | reinterpret_cast<uintptr_t>(p.lam) |
                      reinterpret_cast<uintptr_t>(p.wl) | reinterpret_cast<uintptr_t>(p.wm) |
                      reinterpret_cast<uintptr_t>(p.wr) | reinterpret_cast<uintptr_t>(bwd ? p.dh : p.hout) |
                      reinterpret_cast<uintptr_t>(bwd ? p.h : p.hout) | reinterpret_cast<uintptr_t>(bwd ? p.dlam : p.hout) |
                      reinterpret_cast<uintptr_t>(bwd ? p.dx : p.hout);
  if ((a & 15u) != 0) return false;
  if (p.B * p.G * p.D >= (int64_t{1} << 31)) return false;
  const int kb = cl_batch(p, es, bwd);
  if (kb <= 0) return false;
  // backward: every batch synchronises the cluster (dx needs all D directions); measured on 28 x 28 planes
  // this beats the one-CTA-per-unit kernel only while a unit is at most two batches (configs[2] primary,
  // C_proxy = 8: 32 -> 41 us per step; 48 channels per group: 0.95 vs 0.68 ms), so larger groups stay there
  if (bwd && (p.C / p.G + kb - 1) / kb > 2) return false;
  return true;
}

cudaError_t launch_fwd_small_cl(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches) {
  *launches += 1;
  const int es = dt == GSPN_BF16 ? 2 : 4, kb = cl_batch(p, es, false);
  const size_t smem = cl_layout(static_cast<int>(p.H * p.W), es, kb, 2, 0).total;
  const int threads = (kFwdWarps + 1) * 32;
  const bool local = p.kchunk > 0;
  if (dt == GSPN_BF16)
    return local ? launch_cl(fwd_grp_cl_kernel<__nv_bfloat16, true>, p, threads, kb, smem, s)
                 : launch_cl(fwd_grp_cl_kernel<__nv_bfloat16, false>, p, threads, kb, smem, s);
  return local ? launch_cl(fwd_grp_cl_kernel<float, true>, p, threads, kb, smem, s)
               : launch_cl(fwd_grp_cl_kernel<float, false>, p, threads, kb, smem, s);
}

cudaError_t launch_bwd_small_cl(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches) {
  *launches += 1;
  const int es = dt == GSPN_BF16 ? 2 : 4;
  const int HW = static_cast<int>(p.H * p.W);
  const int64_t Cg = p.C / p.G;
  // a unit of <= 2 kBwdWarps channels: one batch, two chains per warp, one buffer (3a: 8 channels)
  const bool two = Cg <= 2 * kBwdWarps && cl_batch(p, es, true, 2) >= Cg && !knob_set_cl("GSPN_CL_KC1");
  const int kb = two ? static_cast<int>(Cg) : cl_batch(p, es, true, 1);
  const size_t smem = cl_layout(HW, es, kb, 4, static_cast<uint32_t>(kBwdWarps * 3 * HW * 4), two ? 1 : 2).total;
  const int threads = (kBwdWarps + 1) * 32;
  const bool local = p.kchunk > 0;
  using BF = __nv_bfloat16;
  if (two) {
    if (dt == GSPN_BF16)
      return local ? launch_cl(bwd_grp_cl_kernel<BF, true, 2>, p, threads, kb, smem, s)
                   : launch_cl(bwd_grp_cl_kernel<BF, false, 2>, p, threads, kb, smem, s);
    return local ? launch_cl(bwd_grp_cl_kernel<float, true, 2>, p, threads, kb, smem, s)
                 : launch_cl(bwd_grp_cl_kernel<float, false, 2>, p, threads, kb, smem, s);
  }
  if (dt == GSPN_BF16)
    return local ? launch_cl(bwd_grp_cl_kernel<BF, true, 1>, p, threads, kb, smem, s)
                 : launch_cl(bwd_grp_cl_kernel<BF, false, 1>, p, threads, kb, smem, s);
  return local ? launch_cl(bwd_grp_cl_kernel<float, true, 1>, p, threads, kb, smem, s)
               : launch_cl(bwd_grp_cl_kernel<float, false, 1>, p, threads, kb, smem, s);
}

}  // namespace gspn
