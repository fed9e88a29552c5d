// gspn_small.cu — small-plane path (max(H, W) <= 32): the compact-channel and proxy-space shapes of the
// paper (28 x 28 stages with C_proxy channels) whose rows are too short for TMA's
// 16-byte row strides (W s % 16 != 0, e.g. 28 x 2 bytes). SURVEY.md §8(a) a2 "small-plane path".
//
// One CTA per (b, c) plane, one warp per direction (D <= 4 warps). Every plane the chain set needs is
// staged whole in shared memory with coalesced vector loads (a plane is at most 32 x 32 elements); then
// each warp runs its direction's L-step recurrence with lane = position (P <= 32), neighbours by warp
// shuffle, no block barriers inside the scan; outputs leave shared memory with coalesced stores.
// Forward: h_t[r] = a h_{t-1}[r-1] + b h_{t-1}[r] + c h_{t-1}[r+1] + lam x (Eq. 1/3).
// Backward: each warp runs the adjoint recurrence of its direction into an fp32
// g plane; then all threads form, per pixel, dlam_d = g_d x, dx = sum_d g_d lam_d (fixed order, no
// atomics), Da/Db/Dc from h_{t-1} and the normalisation Jacobian -- written directly for per-channel
// weights (G = C), or summed over the group's channels with fp32 red.global.add into the workspace and
// finished by the generic path's finish_dw kernel (G < C).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "gspn_common.cuh"
#include "gspn_internal.h"

namespace gspn {
namespace {

constexpr int kSmallMax = 32;

// Experiment knob (A/B tooling): read only when GSPN_EXPERIMENTS is set.
bool knob_set(const char* name) {
  static const bool on = getenv("GSPN_EXPERIMENTS") != nullptr;
  return on && getenv(name) != nullptr;
}

// Copy n elements (one plane) global -> shared; 16-byte vectors when both sides allow it.
template <typename T>
__device__ __forceinline__ void plane_in(T* dst, const T* src, int n) {
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0 &&
                   (n * static_cast<int>(sizeof(T))) % 16 == 0;
  if (vec) {
    const int nv = n * static_cast<int>(sizeof(T)) / 16;
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    for (int i = threadIdx.x; i < nv; i += blockDim.x) d[i] = __ldg(s + i);
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  }
}

template <typename T>
__device__ __forceinline__ void plane_out(T* dst, const T* src, int n) {
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0 &&
                   (n * static_cast<int>(sizeof(T))) % 16 == 0;
  if (vec) {
    const int nv = n * static_cast<int>(sizeof(T)) / 16;
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    for (int i = threadIdx.x; i < nv; i += blockDim.x) d[i] = s[i];
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  }
}

// Row-normalised taps with the hardware reciprocal (rcp.approx, <= 1 ulp; R15) -- the scan is
// a serial chain per warp, so the IEEE reciprocal's slow-path branch would sit on its critical path.
__device__ __forceinline__ Taps fast_taps(float wl, float wm, float wr, bool has_l, bool has_r, bool prenorm) {
  Taps t;
  const float l = has_l ? wl : 0.f, r = has_r ? wr : 0.f;
  if (prenorm) {
    t.a = l; t.b = wm; t.c = r; t.inv = 1.f;
  } else {
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.inv) : "f"(wm + l + r));
    t.a = l * t.inv; t.b = wm * t.inv; t.c = r * t.inv;
  }
  return t;
}

// Shared-memory planes are padded to 16 bytes so every plane starts aligned.
__host__ __device__ __forceinline__ int padded(int n, int es) { return (n * es + 15) / 16 * 16 / es; }

// Forward. smem: x | per direction: lam, w_l, w_m, w_r, h.
template <typename T, bool kLocal>
__global__ void __launch_bounds__(128) fwd_small_kernel(ScanParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int H = static_cast<int>(p.H), W = static_cast<int>(p.W), HW = H * W, D = static_cast<int>(p.D);
  const int np = padded(HW, sizeof(T));
  const int C32 = static_cast<int>(p.C), Cg32 = static_cast<int>(p.C / p.G);
  const int bc32 = blockIdx.x, b32 = bc32 / C32, c32 = bc32 - b32 * C32;  // 32-bit: B C < 2^31
  const int64_t bc = bc32, b = b32, c = c32, g = c32 / Cg32;
  T* xs = reinterpret_cast<T*>(sm);
  plane_in(xs, static_cast<const T*>(p.x) + bc * HW, HW);
  for (int k = 0; k < D; ++k) {
    T* base = xs + np * (1 + 5 * k);
    const int64_t chain = (k * p.B + b) * p.C + c, wpl = (k * p.B + b) * p.G + g;
    plane_in(base, static_cast<const T*>(p.lam) + chain * HW, HW);
    plane_in(base + np, static_cast<const T*>(p.wl) + wpl * HW, HW);
    plane_in(base + 2 * np, static_cast<const T*>(p.wm) + wpl * HW, HW);
    plane_in(base + 3 * np, static_cast<const T*>(p.wr) + wpl * HW, HW);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, r = threadIdx.x & 31;
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  if (warp < D) {
    const uint32_t dir = p.dirbit[warp];
    const DirGeom gm = dir_geom(dir, H, W);
    const int L = static_cast<int>(gm.L), P = static_cast<int>(gm.P);
    const int gbase = static_cast<int>(gm.base), gts = static_cast<int>(gm.ts), grs = static_cast<int>(gm.rs);
    const int kc = static_cast<int>(p.kchunk);
    const T* lam = xs + np * (1 + 5 * warp);
    const T *wl = lam + np, *wm = lam + 2 * np, *wr = lam + 3 * np;
    T* h = xs + np * (1 + 5 * warp) + 4 * np;
    const bool in = r < P, hl = r >= 1, hr = r <= P - 2;
    float hv = 0.f;
    int off = gbase + (in ? r : 0) * grs;
    for (int t = 0; t < L; ++t, off += gts) {
      if constexpr (kLocal) {
        if (seg_start_step(dir, t, L, kc)) hv = 0.f;  // warp-uniform: h_{t-1} does not propagate
      }
      const float up = __shfl_up_sync(0xffffffffu, hv, 1);
      const float dn = __shfl_down_sync(0xffffffffu, hv, 1);
      // masked taps are 0: lanes outside [0, P) (hv = 0) and the shuffle wrap never couple in
      const Taps tp = fast_taps(to_f(wl[off]), to_f(wm[off]), to_f(wr[off]), hl, hr, prenorm);
      const float v = fmaf(tp.a, up, fmaf(tp.b, hv, fmaf(tp.c, dn, to_f(lam[off]) * to_f(xs[off]))));
      if (in) h[off] = from_f<T>(v);
      hv = in ? v : 0.f;
    }
  }
  __syncthreads();
  for (int k = 0; k < D; ++k) {
    const int64_t chain = (k * p.B + b) * p.C + c;
    plane_out(static_cast<T*>(p.hout) + chain * HW, xs + np * (1 + 5 * k + 4), HW);
  }
}

// Backward. smem: x | per direction: lam, w_l, w_m, w_r, h, dh | fp32 g planes [D][HW].
template <typename T, bool kPerChannel, bool kLocal>
__global__ void __launch_bounds__(128) bwd_small_kernel(ScanParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int H = static_cast<int>(p.H), W = static_cast<int>(p.W), HW = H * W, D = static_cast<int>(p.D);
  const int np = padded(HW, sizeof(T));
  const int C32 = static_cast<int>(p.C), Cg32 = static_cast<int>(p.C / p.G);
  const int bc32 = blockIdx.x, b32 = bc32 / C32, c32 = bc32 - b32 * C32;
  const int64_t bc = bc32, b = b32, c = c32, g = c32 / Cg32;
  T* xs = reinterpret_cast<T*>(sm);
  float* gs = reinterpret_cast<float*>(sm + static_cast<size_t>(np) * (1 + 6 * D) * sizeof(T));
  plane_in(xs, static_cast<const T*>(p.x) + bc * HW, HW);
  for (int k = 0; k < D; ++k) {
    T* base = xs + np * (1 + 6 * k);
    const int64_t chain = (k * p.B + b) * p.C + c, wpl = (k * p.B + b) * p.G + g;
    plane_in(base, static_cast<const T*>(p.lam) + chain * HW, HW);
    plane_in(base + np, static_cast<const T*>(p.wl) + wpl * HW, HW);
    plane_in(base + 2 * np, static_cast<const T*>(p.wm) + wpl * HW, HW);
    plane_in(base + 3 * np, static_cast<const T*>(p.wr) + wpl * HW, HW);
    plane_in(base + 4 * np, static_cast<const T*>(p.h) + chain * HW, HW);
    plane_in(base + 5 * np, static_cast<const T*>(p.dh) + chain * HW, HW);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, r = threadIdx.x & 31;
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  if (warp < D) {  // adjoint recurrence, reverse step order: g_t = dh_t + (b g)[r] + (a g)[r+1] + (c g)[r-1]
    const uint32_t dir = p.dirbit[warp];
    const DirGeom gm = dir_geom(dir, H, W);
    const int L = static_cast<int>(gm.L), P = static_cast<int>(gm.P);
    const int gbase = static_cast<int>(gm.base), gts = static_cast<int>(gm.ts), grs = static_cast<int>(gm.rs);
    const int kc = static_cast<int>(p.kchunk);
    const T* lam = xs + np * (1 + 6 * warp);
    const T *wl = lam + np, *wm = lam + 2 * np, *wr = lam + 3 * np, *dh = lam + 5 * np;
    float* gp = gs + warp * HW;
    const bool in = r < P, hl = r >= 1, hr = r <= P - 2;
    float ea = 0.f, eb = 0.f, ec = 0.f;  // (a g, b g, c g) of step t+1 at this position
    int off = gbase + (L - 1) * gts + (in ? r : 0) * grs;
    for (int t = L - 1; t >= 0; --t, off -= gts) {
      const float from_r = __shfl_down_sync(0xffffffffu, ea, 1);  // a_{t+1}[r+1] g_{t+1}[r+1]
      const float from_l = __shfl_up_sync(0xffffffffu, ec, 1);    // c_{t+1}[r-1] g_{t+1}[r-1]
      // lanes outside [0, P) carry 0; the masks stop the shuffle wrap at lanes 0 / 31
      const float gt = to_f(dh[off]) + eb + ((hr ? from_r : 0.f) + (hl ? from_l : 0.f));
      if (in) gp[off] = gt;
      const Taps tp = fast_taps(to_f(wl[off]), to_f(wm[off]), to_f(wr[off]), hl, hr, prenorm);
      const float gi = in ? gt : 0.f;
      ea = tp.a * gi; eb = tp.b * gi; ec = tp.c * gi;
      if constexpr (kLocal) {
        if (seg_start_step(dir, t, L, kc)) ea = eb = ec = 0.f;  // h_t did not depend on h_{t-1}
      }
    }
  }
  __syncthreads();
  // per pixel: dlam_d, dx, and the tap gradients of every direction
  for (int px = threadIdx.x; px < HW; px += blockDim.x) {
    const int i = px / W, j = px - (px / W) * W;
    const float xv = to_f(xs[px]);
    float dx = 0.f;
    for (int k = 0; k < D; ++k) {
      const T* lam = xs + np * (1 + 6 * k);
      const T *wl = lam + np, *wm = lam + 2 * np, *wr = lam + 3 * np, *h = lam + 4 * np;
      const float gt = gs[k * HW + px];
      const int64_t chain = (k * p.B + b) * p.C + c;
      static_cast<T*>(p.dlam)[chain * HW + px] = from_f<T>(gt * xv);
      dx = fmaf(gt, to_f(lam[px]), dx);
      const uint32_t dir = p.dirbit[k];
      const bool vert = is_vertical(dir);
      const int t = dir == GSPN_DIR_T2B ? i : dir == GSPN_DIR_B2T ? H - 1 - i : dir == GSPN_DIR_L2R ? j : W - 1 - j;
      const int L = vert ? H : W, P = vert ? W : H, rr = vert ? j : i;
      const bool hl = rr >= 1, hr = rr <= P - 2;
      float Da = 0.f, Db = 0.f, Dc = 0.f;
      if (!seg_start_step(dir, t, L, static_cast<int>(p.kchunk))) {  // h_{t-1} and its neighbours along the parallel axis
        const int prev = dir == GSPN_DIR_T2B ? px - W : dir == GSPN_DIR_B2T ? px + W : dir == GSPN_DIR_L2R ? px - 1 : px + 1;
        const int rs = vert ? 1 : W;
        Db = gt * to_f(h[prev]);
        if (hl) Da = gt * to_f(h[prev - rs]);
        if (hr) Dc = gt * to_f(h[prev + rs]);
      }
      const int64_t wofs = ((k * p.B + b) * p.G + g) * HW + px;
      if constexpr (kPerChannel) {
        float ol, om, orr;
        jacobian<true>(to_f(wl[px]), to_f(wm[px]), to_f(wr[px]), hl, hr, prenorm, Da, Db, Dc, ol, om, orr);
        static_cast<T*>(p.dwl)[wofs] = from_f<T>(hl ? ol : 0.f);
        static_cast<T*>(p.dwm)[wofs] = from_f<T>(om);
        static_cast<T*>(p.dwr)[wofs] = from_f<T>(hr ? orr : 0.f);
      } else {
        if (hl) atomicAdd(p.dwa_l + wofs, Da);
        atomicAdd(p.dwa_m + wofs, Db);
        if (hr) atomicAdd(p.dwa_r + wofs, Dc);
      }
    }
    static_cast<T*>(p.dx)[bc * HW + px] = from_f<T>(dx);
  }
}

// ---------------------------------------------------------------------------------------------------
// Grouped weights (G < C: configs 3a / 3b, the compact-channel variant of PAPER.md:140-148 Eq. 3).
// One CTA per unit (b, g). The normalised taps of every direction are computed ONCE per (d, b, g, t, r)
// into shared memory (fp32, scan order, so lane r of every direction reads consecutive words) and
// reused by all C/G channels of the group -- the per-channel re-normalisation of
// the per-plane kernels above is gone. Warps take the group's channels in turn; a warp stages its
// channel's x plane once and runs the D directions on it (lane = position, neighbours by shuffle), its
// lam / h / dh planes staged whole with 16-byte vectors and written back the same way.
// Backward: see bwd_grp_small_kernel (dlam in place over the dh plane; dx and the group sums reduced in a
// fixed order -- bitwise deterministic); the Jacobian and the dw stores follow once per unit.
constexpr int kGrpWarpsF = 12, kGrpWarpsB = 8;

// One plane (<= 32 x 32 elements) global -> shared by one warp: every 16-byte load is issued before the
// first store, so the warp waits for one memory latency, not one per vector.
template <typename T>
__device__ __forceinline__ void warp_plane_in(T* dst, const T* src, int n, int lane) {
  constexpr int kV = kSmallMax * kSmallMax * static_cast<int>(sizeof(T)) / 16 / 32;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0 &&
      (n * static_cast<int>(sizeof(T))) % 16 == 0) {
    const int nv = n * static_cast<int>(sizeof(T)) / 16;
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    uint4 v[kV];
#pragma unroll
    for (int i = 0; i < kV; ++i)
      if (lane + 32 * i < nv) v[i] = __ldg(s + lane + 32 * i);
#pragma unroll
    for (int i = 0; i < kV; ++i)
      if (lane + 32 * i < nv) d[lane + 32 * i] = v[i];
  } else {
    for (int i = lane; i < n; i += 32) dst[i] = src[i];
  }
}

template <typename T>
__device__ __forceinline__ void warp_plane_out(T* dst, const T* src, int n, int lane) {
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0 &&
      (n * static_cast<int>(sizeof(T))) % 16 == 0) {
    const int nv = n * static_cast<int>(sizeof(T)) / 16;
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    for (int i = lane; i < nv; i += 32) d[i] = s[i];
  } else {
    for (int i = lane; i < n; i += 32) dst[i] = src[i];
  }
}

// Normalised taps of unit (b, g), all directions: TP[k HW + t P + r] = (a, b, c, 0) (DESIGN.md
// R1/R2), one 16-byte read per lane and step.
template <typename T>
__device__ void unit_taps(const ScanParams& p, int64_t b, int64_t g, float4* TP) {
  const int H = static_cast<int>(p.H), W = static_cast<int>(p.W), HW = H * W, D = static_cast<int>(p.D);
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  for (int idx = threadIdx.x; idx < D * HW; idx += blockDim.x) {
    const int k = idx / HW, q = idx - k * HW;
    const DirGeom gm = dir_geom(p.dirbit[k], H, W);
    const int P = static_cast<int>(gm.P), t = q / P, r = q - t * P;
    const int pix = static_cast<int>(gm.base + t * gm.ts + r * gm.rs);
    const int64_t w = ((k * p.B + b) * p.G + g) * HW + pix;
    const Taps tp = make_taps(to_f(static_cast<const T*>(p.wl)[w]), to_f(static_cast<const T*>(p.wm)[w]),
                              to_f(static_cast<const T*>(p.wr)[w]), r >= 1, r <= P - 2, prenorm);
    TP[idx] = make_float4(tp.a, tp.b, tp.c, 0.f);
  }
}

__device__ __forceinline__ void named_barrier(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__host__ __device__ __forceinline__ size_t align16(size_t v) { return (v + 15) / 16 * 16; }

// A whole plane (<= 32 x 32) held in registers as 16-byte vectors, kV per lane: loaded while the warp
// computes the previous plane (software pipelining of the staging), stored to shared memory after.
template <typename T>
struct PlaneRegs {
  static constexpr int kV = kSmallMax * kSmallMax * static_cast<int>(sizeof(T)) / 16 / 32;
  uint4 v[kV];
  __device__ __forceinline__ void load(const T* src, int n, int lane, bool vec) {
    if (!vec) return;
    const uint4* s = reinterpret_cast<const uint4*>(src);
    const int nv = n * static_cast<int>(sizeof(T)) / 16;
#pragma unroll
    for (int i = 0; i < kV; ++i)
      if (lane + 32 * i < nv) v[i] = __ldg(s + lane + 32 * i);
  }
  __device__ __forceinline__ void store(T* dst, const T* src, int n, int lane, bool vec) const {
    if (!vec) {  // unaligned plane size: plain element copy
      for (int i = lane; i < n; i += 32) dst[i] = src[i];
      return;
    }
    uint4* d = reinterpret_cast<uint4*>(dst);
    const int nv = n * static_cast<int>(sizeof(T)) / 16;
#pragma unroll
    for (int i = 0; i < kV; ++i)
      if (lane + 32 * i < nv) d[lane + 32 * i] = v[i];
  }
};

template <typename T>
__device__ __forceinline__ bool plane_vec(const ScanParams& p) {
  // every plane of every tensor starts 16-byte aligned and is a whole number of 16-byte vectors
  const uintptr_t a = reinterpret_cast<uintptr_t>(p.x) | reinterpret_cast<uintptr_t>(p.lam) |
                      reinterpret_cast<uintptr_t>(p.h) | reinterpret_cast<uintptr_t>(p.dh) |
                      reinterpret_cast<uintptr_t>(p.hout) | reinterpret_cast<uintptr_t>(p.dlam);
  return (a & 15u) == 0 && (p.H * p.W * static_cast<int64_t>(sizeof(T))) % 16 == 0;
}

template <typename T, bool kLocal>
__global__ void __launch_bounds__(kGrpWarpsF * 32, 2) fwd_grp_small_kernel(ScanParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int H = static_cast<int>(p.H), W = static_cast<int>(p.W), HW = H * W, D = static_cast<int>(p.D);
  const int np = padded(HW, sizeof(T));
  const int64_t G = p.G, Cg = p.C / p.G;
  const int64_t b = blockIdx.x / G, g = blockIdx.x % G;
  float4* TP = reinterpret_cast<float4*>(sm);
  T* wbuf = reinterpret_cast<T*>(sm + static_cast<size_t>(D * HW) * 16);
  const bool vec = plane_vec<T>(p);
  unit_taps<T>(p, b, g, TP);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  T* X = wbuf + static_cast<size_t>(warp) * 2 * np;
  T* Lm = X + np;
  const int kc = static_cast<int>(p.kchunk);
  const T* lam_g = static_cast<const T*>(p.lam);
  // items (channel cc, direction k) of this warp, in order; lam of the next item is prefetched
  const int64_t nitems = ((Cg - warp + nw - 1) / nw) * D;
  auto chain_of = [&](int64_t it) {
    const int64_t cc = warp + (it / D) * nw;
    return ((it % D) * p.B + b) * p.C + g * Cg + cc;
  };
  PlaneRegs<T> pre;
  if (nitems > 0) pre.load(lam_g + chain_of(0) * HW, HW, lane, vec);
  __syncthreads();  // taps ready
  for (int64_t it = 0; it < nitems; ++it) {
    const int k = static_cast<int>(it % D);
    const int64_t cc = warp + (it / D) * nw;
    const int64_t c = g * Cg + cc;
    const int64_t chain = chain_of(it);
    if (k == 0) {  // a new channel: its x plane, shared by the D directions
      __syncwarp();
      warp_plane_in(X, static_cast<const T*>(p.x) + (b * p.C + c) * HW, HW, lane);
    }
    pre.store(Lm, lam_g + chain * HW, HW, lane, vec);
    if (it + 1 < nitems) pre.load(lam_g + chain_of(it + 1) * HW, HW, lane, vec);
    __syncwarp();
    const uint32_t dir = p.dirbit[k];
    const DirGeom gm = dir_geom(dir, H, W);
    const int L = static_cast<int>(gm.L), P = static_cast<int>(gm.P);
    const int ts = static_cast<int>(gm.ts);
    const bool in = lane < P;
    const int r = in ? lane : 0;
    const float4* tq = TP + k * HW + r;
    const int off0 = static_cast<int>(gm.base) + r * static_cast<int>(gm.rs);
    const T* xp = X + off0;
    T* lp = Lm + off0;
    float hv = 0.f;
#pragma unroll 4
    for (int t = 0; t < L; ++t) {
      if constexpr (kLocal) {
        if (seg_start_step(dir, t, L, kc)) hv = 0.f;  // warp-uniform: h_{t-1} does not propagate
      }
      const float up = __shfl_up_sync(0xffffffffu, hv, 1);    // lane 0: tap a = 0
      const float dn = __shfl_down_sync(0xffffffffu, hv, 1);  // lane P-1: tap c = 0; lanes >= P carry 0
      const float4 q = *tq;
      // lanes >= P read x instead of lam: x is never written, lam at position 0 is (by lane 0)
      const float v = fmaf(q.x, up, fmaf(q.y, hv, fmaf(q.z, dn, to_f(in ? *lp : *xp) * to_f(*xp))));
      if (in) *lp = from_f<T>(v);  // h over lam at the lane's own pixel (neighbours travel by shuffle)
      hv = in ? v : 0.f;
      tq += P;
      xp += ts;
      lp += ts;
    }
    __syncwarp();
    warp_plane_out(static_cast<T*>(p.hout) + chain * HW, Lm, HW, lane);
  }
}

// Backward, grouped weights. Warps form `nslot` slots of D warps; warp (slot j, k) runs direction k on the
// channels j, j + nslot, ... of the group, so the D directions of a channel run side by side. Per channel a
// slot shares the x plane, each warp writes g_k lam_k into its own fp32 plane, and after a slot barrier the
// slot sums those planes in direction order into dx (no atomics, fixed order). The tap-gradient group sums
// of a warp's direction accumulate in its own fp32 partial planes (scan order, lane r owns position r)
// across all its channels; the slots' partials are added in slot order after the channel loop. Every
// reduction has a fixed order: the backward is bitwise deterministic.
template <typename T, bool kLocal>
__global__ void __launch_bounds__(kGrpWarpsB * 32, 1) bwd_grp_small_kernel(ScanParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int H = static_cast<int>(p.H), W = static_cast<int>(p.W), HW = H * W, D = static_cast<int>(p.D);
  const int np = padded(HW, sizeof(T));
  const int64_t G = p.G, Cg = p.C / p.G;
  const int64_t b = blockIdx.x / G, g = blockIdx.x % G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nslot = nw / D, k = warp % D, slot = warp / D;
  float4* TP = reinterpret_cast<float4*>(sm);
  uint8_t* sb = sm + align16(static_cast<size_t>(D * HW) * 16);
  const size_t xb = align16(static_cast<size_t>(np) * sizeof(T));
  const size_t pl_b = align16(3 * static_cast<size_t>(np) * sizeof(T));  // lam, dh, h planes
  const size_t pk_b = align16(static_cast<size_t>(HW) * 4);              // g_k lam_k (fp32)
  const size_t per_warp = pl_b + 4 * pk_b;                               // + partial Da / Db / Dc
  const size_t per_slot = xb + D * per_warp;
  T* X = reinterpret_cast<T*>(sb + slot * per_slot);
  uint8_t* wbase = sb + slot * per_slot + xb;
  uint8_t* mine = wbase + k * per_warp;
  T* Lm = reinterpret_cast<T*>(mine);
  T* DH = Lm + np;
  T* Hs = DH + np;
  float* Pk = reinterpret_cast<float*>(mine + pl_b);
  float* SA = reinterpret_cast<float*>(mine + pl_b + pk_b);  // partial group sums, [t P + r]
  float* SB = SA + pk_b / 4;
  float* SC = SB + pk_b / 4;
  unit_taps<T>(p, b, g, TP);
  for (int i = lane; i < HW; i += 32) SA[i] = SB[i] = SC[i] = 0.f;
  __syncthreads();
  const int kc = static_cast<int>(p.kchunk);
  const uint32_t dir = p.dirbit[k];
  const DirGeom gm = dir_geom(dir, H, W);
  const int L = static_cast<int>(gm.L), P = static_cast<int>(gm.P);
  const int ts = static_cast<int>(gm.ts), rs = static_cast<int>(gm.rs);
  const bool in = lane < P;
  const int r = in ? lane : 0;
  const bool hl = in && r >= 1, hr = in && r <= P - 2;
  const int dl = hl ? -rs : 0, dr = hr ? rs : 0;  // h_{t-1} neighbour offsets (clamped in range)
  const int off_r = static_cast<int>(gm.base) + r * rs;
  const int nch = static_cast<int>((Cg - slot + nslot - 1) / nslot);
  const int bar_id = 1 + slot, bar_n = D * 32;
  const bool vec = plane_vec<T>(p);
  const T *x_g = static_cast<const T*>(p.x), *lam_g = static_cast<const T*>(p.lam);
  const T *dh_g = static_cast<const T*>(p.dh), *h_g = static_cast<const T*>(p.h);
  auto chan = [&](int i) { return g * Cg + slot + static_cast<int64_t>(i) * nslot; };
  PlaneRegs<T> px_, pl_, pd_, ph_;  // the next channel's planes, loaded during this channel's recurrence
  if (nch > 0) {
    const int64_t c0 = chan(0), cb = (b * p.C + c0) * HW, ck = ((k * p.B + b) * p.C + c0) * HW;
    if (k == 0) px_.load(x_g + cb, HW, lane, vec);
    pl_.load(lam_g + ck, HW, lane, vec);
    pd_.load(dh_g + ck, HW, lane, vec);
    ph_.load(h_g + ck, HW, lane, vec);
  }
  for (int i = 0; i < nch; ++i) {
    const int64_t c = chan(i);
    const int64_t bc = b * p.C + c;
    const int64_t chain = (k * p.B + b) * p.C + c;
    if (k == 0) px_.store(X, x_g + bc * HW, HW, lane, vec);
    pl_.store(Lm, lam_g + chain * HW, HW, lane, vec);
    pd_.store(DH, dh_g + chain * HW, HW, lane, vec);
    ph_.store(Hs, h_g + chain * HW, HW, lane, vec);
    if (i + 1 < nch) {
      const int64_t cn = chan(i + 1), cb = (b * p.C + cn) * HW, ck = ((k * p.B + b) * p.C + cn) * HW;
      if (k == 0) px_.load(x_g + cb, HW, lane, vec);
      pl_.load(lam_g + ck, HW, lane, vec);
      pd_.load(dh_g + ck, HW, lane, vec);
      ph_.load(h_g + ck, HW, lane, vec);
    }
    named_barrier(bar_id, bar_n);  // x staged; the previous channel's dx has read every Pk
    float ea = 0.f, eb = 0.f, ec = 0.f;  // (a g, b g, c g) of step t+1 at this position
    // one pointer per array, stepped by -ts (pixels) / -P (scan order): no per-access address arithmetic
    const int off0 = off_r + (L - 1) * ts, q0 = (L - 1) * P + r;
    T* dhp = DH + off0;
    const T* xp = X + off0;
    const T* lp = Lm + off0;
    const T* hp = Hs + off0 - ts;  // h_{t-1} at (t-1, r)
    float* pkp = Pk + off0;
    float* sap = SA + q0;
    float* sbp = SB + q0;
    float* scp = SC + q0;
    const float4* tq = TP + k * HW + q0;
#pragma unroll 2
    for (int t = L - 1; t >= 0; --t) {
      const float from_r = __shfl_down_sync(0xffffffffu, ea, 1);  // a_{t+1}[r+1] g_{t+1}[r+1]
      const float from_l = __shfl_up_sync(0xffffffffu, ec, 1);    // c_{t+1}[r-1] g_{t+1}[r-1]
      // lanes >= P alias position 0: they read only arrays nobody writes (x, the taps), so lane 0's
      // in-place writes below never race with them
      const float gsum = to_f(in ? *dhp : *xp) + eb + ((hr ? from_r : 0.f) + (hl ? from_l : 0.f));
      const float gt = in ? gsum : 0.f;
      const float4 tp = *tq;
      const bool seg = seg_start_step(dir, t, L, kc);  // warp-uniform; t = 0 always: h_{-1} = 0
      const float gh = seg ? 0.f : gt;
      const T* hq = seg ? xp : hp;  // any in-plane pixel when h_{t-1} is not used (t = 0: hp is off-plane)
      const float* ro = reinterpret_cast<const float*>(tq);  // read-only stand-in for lanes >= P
      const float sb_ = fmaf(gh, to_f(hq[0]), in ? *sbp : *ro);
      const float sa_ = fmaf(hl ? gh : 0.f, to_f(hq[dl]), in ? *sap : *ro);
      const float sc_ = fmaf(hr ? gh : 0.f, to_f(hq[dr]), in ? *scp : *ro);
      const float dlam = gt * to_f(*xp);
      const float pk = gt * to_f(*lp);
      if (in) {
        *dhp = from_f<T>(dlam);  // dlam over dh (read above)
        *pkp = pk;               // g_k lam_k, summed over k into dx below
        *sap = sa_;
        *sbp = sb_;
        *scp = sc_;
      }
      ea = tp.x * gt;
      eb = tp.y * gt;
      ec = tp.z * gt;
      if constexpr (kLocal) {
        if (seg) ea = eb = ec = 0.f;  // h_t did not depend on h_{t-1}
      }
      dhp -= ts; xp -= ts; lp -= ts; hp -= ts; pkp -= ts;
      sap -= P; sbp -= P; scp -= P; tq -= P;
    }
    __syncwarp();
    warp_plane_out(static_cast<T*>(p.dlam) + chain * HW, DH, HW, lane);
    named_barrier(bar_id, bar_n);  // every direction's g lam of this channel is in its Pk
    T* dxo = static_cast<T*>(p.dx) + bc * HW;
    for (int px = k * 32 + lane; px < HW; px += bar_n) {
      float acc = 0.f;
      for (int kk = 0; kk < D; ++kk) acc += reinterpret_cast<const float*>(wbase + kk * per_warp + pl_b)[px];
      dxo[px] = from_f<T>(acc);
    }
  }
  __syncthreads();
  // dw = normalisation Jacobian of the group sums (slot partials added in slot order)
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  const bool f32out = p.flags & GSPN_FLAG_DW_F32;
  for (int idx = threadIdx.x; idx < D * HW; idx += blockDim.x) {
    const int kk = idx / HW, q = idx - kk * HW;
    const DirGeom gk = dir_geom(p.dirbit[kk], H, W);
    const int Pq = static_cast<int>(gk.P), t = q / Pq, rr = q - t * Pq;
    const int pix = static_cast<int>(gk.base + t * gk.ts + rr * gk.rs);
    const int64_t w = ((kk * p.B + b) * p.G + g) * HW + pix;
    float Da = 0.f, Db = 0.f, Dc = 0.f;
    for (int j = 0; j < nslot; ++j) {
      const float* part = reinterpret_cast<const float*>(sb + j * per_slot + xb + kk * per_warp + pl_b + pk_b);
      Da += part[q];
      Db += part[pk_b / 4 + q];
      Dc += part[2 * (pk_b / 4) + q];
    }
    const bool l_on = rr >= 1, r_on = rr <= Pq - 2;
    float ol, om, orr;
    jacobian(to_f(static_cast<const T*>(p.wl)[w]), to_f(static_cast<const T*>(p.wm)[w]),
             to_f(static_cast<const T*>(p.wr)[w]), l_on, r_on, prenorm, Da, Db, Dc, ol, om, orr);
    if (f32out) {
      static_cast<float*>(p.dwl)[w] = ol;
      static_cast<float*>(p.dwm)[w] = om;
      static_cast<float*>(p.dwr)[w] = orr;
    } else {
      static_cast<T*>(p.dwl)[w] = from_f<T>(ol);
      static_cast<T*>(p.dwm)[w] = from_f<T>(om);
      static_cast<T*>(p.dwr)[w] = from_f<T>(orr);
    }
  }
}

size_t grp_fwd_smem(const ScanParams& p, int es, int nw) {
  const int np = padded(static_cast<int>(p.H * p.W), es);
  return static_cast<size_t>(p.D * p.H * p.W) * 16 + static_cast<size_t>(nw) * 2 * np * es;
}
size_t grp_bwd_smem(const ScanParams& p, int es, int nw) {
  const int np = padded(static_cast<int>(p.H * p.W), es);
  const size_t HW = static_cast<size_t>(p.H * p.W), D = static_cast<size_t>(p.D);
  const size_t per_warp = align16(3 * static_cast<size_t>(np) * es) + 4 * align16(HW * 4);
  const size_t per_slot = align16(static_cast<size_t>(np) * es) + D * per_warp;
  return align16(D * HW * 16) + static_cast<size_t>(nw / p.D) * per_slot;
}

template <typename K>
cudaError_t launch_grp(K kern, const ScanParams& p, int nw, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<static_cast<unsigned>(p.B * p.G), nw * 32, smem, s>>>(p);
  return cudaGetLastError();
}

// warps per CTA: no more than the group has channels, and within the shared-memory budget
int grp_warps(const ScanParams& p, int es, bool bwd) {
  const int64_t Cg = p.C / p.G;
  const size_t budget = static_cast<size_t>(device_smem_optin());
  if (bwd) {  // D warps per slot, at most one slot per channel
    const int D = static_cast<int>(p.D);
    int ns = static_cast<int>(std::min<int64_t>(kGrpWarpsB / D, Cg));
    while (ns > 1 && grp_bwd_smem(p, es, ns * D) > budget) --ns;
    return grp_bwd_smem(p, es, ns * D) <= budget ? ns * D : 0;
  }
  int nw = static_cast<int>(std::min<int64_t>(kGrpWarpsF, Cg));
  while (nw > 1 && grp_fwd_smem(p, es, nw) > budget) --nw;
  return grp_fwd_smem(p, es, nw) <= budget ? nw : 0;
}

size_t fwd_smem(const ScanParams& p, int es) {
  const int np = padded(static_cast<int>(p.H * p.W), es);
  return static_cast<size_t>(np) * (1 + 5 * p.D) * es;
}
size_t bwd_smem(const ScanParams& p, int es) {
  const int np = padded(static_cast<int>(p.H * p.W), es);
  return static_cast<size_t>(np) * (1 + 6 * p.D) * es + static_cast<size_t>(p.D * p.H * p.W) * 4;
}

template <typename K>
cudaError_t launch_small(K kern, const ScanParams& p, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<static_cast<unsigned>(p.B * p.C), 128, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

bool small_eligible(const ScanParams& p) { return p.H <= kSmallMax && p.W <= kSmallMax && p.D <= 4; }

bool small_grouped(const ScanParams& p, gspn_dtype_t dt) {
  return p.G < p.C && grp_warps(p, dt == GSPN_BF16 ? 2 : 4, true) > 0 && grp_warps(p, dt == GSPN_BF16 ? 2 : 4, false) > 0;
}

cudaError_t launch_fwd_small(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches) {
  if (small_cl_eligible(p, dt, false) && !knob_set("GSPN_NO_SMALL_CL")) return launch_fwd_small_cl(p, dt, s, launches);
  *launches += 1;
  const bool local = p.kchunk > 0;
  if (small_grouped(p, dt)) {
    const int es = dt == GSPN_BF16 ? 2 : 4, nw = grp_warps(p, es, false);
    const size_t sm = grp_fwd_smem(p, es, nw);
    if (dt == GSPN_BF16)
      return local ? launch_grp(fwd_grp_small_kernel<__nv_bfloat16, true>, p, nw, sm, s)
                   : launch_grp(fwd_grp_small_kernel<__nv_bfloat16, false>, p, nw, sm, s);
    return local ? launch_grp(fwd_grp_small_kernel<float, true>, p, nw, sm, s)
                 : launch_grp(fwd_grp_small_kernel<float, false>, p, nw, sm, s);
  }
  if (dt == GSPN_BF16)
    return local ? launch_small(fwd_small_kernel<__nv_bfloat16, true>, p, fwd_smem(p, 2), s)
                 : launch_small(fwd_small_kernel<__nv_bfloat16, false>, p, fwd_smem(p, 2), s);
  return local ? launch_small(fwd_small_kernel<float, true>, p, fwd_smem(p, 4), s)
               : launch_small(fwd_small_kernel<float, false>, p, fwd_smem(p, 4), s);
}

// Grouped weights: the whole backward (dw included) in one launch, no workspace.
cudaError_t launch_bwd_small_grouped(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches) {
  if (small_cl_eligible(p, dt, true) && !knob_set("GSPN_NO_SMALL_CL")) return launch_bwd_small_cl(p, dt, s, launches);
  *launches += 1;
  const bool local = p.kchunk > 0;
  const int es = dt == GSPN_BF16 ? 2 : 4, nw = grp_warps(p, es, true);
  const size_t sm = grp_bwd_smem(p, es, nw);
  if (dt == GSPN_BF16)
    return local ? launch_grp(bwd_grp_small_kernel<__nv_bfloat16, true>, p, nw, sm, s)
                 : launch_grp(bwd_grp_small_kernel<__nv_bfloat16, false>, p, nw, sm, s);
  return local ? launch_grp(bwd_grp_small_kernel<float, true>, p, nw, sm, s)
               : launch_grp(bwd_grp_small_kernel<float, false>, p, nw, sm, s);
}

// Per-plane kernels (G = C directly; G < C only when the grouped kernel does not fit): for G < C p.dwa_*
// must point at zeroed fp32 workspace and the caller then runs the generic finish_dw.
cudaError_t launch_bwd_small(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches) {
  *launches += 1;
  const bool pc = p.G == p.C, lo = p.kchunk > 0;
  using BF = __nv_bfloat16;
  if (dt == GSPN_BF16) {
    if (pc) return lo ? launch_small(bwd_small_kernel<BF, true, true>, p, bwd_smem(p, 2), s)
                      : launch_small(bwd_small_kernel<BF, true, false>, p, bwd_smem(p, 2), s);
    return lo ? launch_small(bwd_small_kernel<BF, false, true>, p, bwd_smem(p, 2), s)
              : launch_small(bwd_small_kernel<BF, false, false>, p, bwd_smem(p, 2), s);
  }
  if (pc) return lo ? launch_small(bwd_small_kernel<float, true, true>, p, bwd_smem(p, 4), s)
                    : launch_small(bwd_small_kernel<float, true, false>, p, bwd_smem(p, 4), s);
  return lo ? launch_small(bwd_small_kernel<float, false, true>, p, bwd_smem(p, 4), s)
            : launch_small(bwd_small_kernel<float, false, false>, p, bwd_smem(p, 4), s);
}

}  // namespace gspn
