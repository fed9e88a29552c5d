// gspn_generic.cu — the generic CUDA path: correct for every shape, dtype and alignment the ABI
// accepts (ragged sizes, H or W = 1, any group count). One CTA per chain (direction, b, c); the
// previous step's hidden state lives in shared memory ("SRAM for hidden states"),
// the whole L-step loop runs inside one launch ("Kernel Fuse"). Loads are direct
// global loads (coalesced for T2B/B2T, strided for L2R/R2L); the TMA streaming path in
// gspn_stream.cu is the fast path for aligned shapes.
#include "gspn_common.cuh"
#include "gspn_internal.h"

namespace gspn {
namespace {

struct ChainIdx {
  int k;          // direction slab
  int64_t bc;     // b * C + c
  int64_t b, c, g;
  int64_t chain;  // (k * B + b) * C + c
};

__device__ __forceinline__ ChainIdx chain_idx(const ScanParams& p, int64_t chain) {
  ChainIdx ci;
  const int64_t BC = p.B * p.C;
  ci.chain = chain;
  ci.k = (int)(chain / BC);
  ci.bc = chain % BC;
  ci.b = ci.bc / p.C;
  ci.c = ci.bc % p.C;
  ci.g = ci.c / (p.C / p.G);
  return ci;
}

// Forward, Eq. 1 / Eq. 3, h_{-1} = 0.
template <typename T>
__global__ void __launch_bounds__(1024) fwd_generic_kernel(ScanParams p) {
  extern __shared__ float smem[];
  const ChainIdx ci = chain_idx(p, blockIdx.x);
  const DirGeom gm = dir_geom(p.dirbit[ci.k], p.H, p.W);
  const int64_t HW = p.H * p.W;
  const T* x = static_cast<const T*>(p.x) + ci.bc * HW;
  const T* lam = static_cast<const T*>(p.lam) + ci.chain * HW;
  const int64_t wofs = ((ci.k * p.B + ci.b) * p.G + ci.g) * HW;
  const T* wl = static_cast<const T*>(p.wl) + wofs;
  const T* wm = static_cast<const T*>(p.wm) + wofs;
  const T* wr = static_cast<const T*>(p.wr) + wofs;
  T* h = static_cast<T*>(p.hout) + ci.chain * HW;
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  float* hp = smem;
  float* hc = smem + gm.P;
  for (int64_t t = 0; t < gm.L; ++t) {
    for (int64_t r = threadIdx.x; r < gm.P; r += blockDim.x) {
      const int64_t off = gm.base + t * gm.ts + r * gm.rs;
      const Taps tp = make_taps(to_f(wl[off]), to_f(wm[off]), to_f(wr[off]), r >= 1, r <= gm.P - 2, prenorm);
      float acc = 0.f;
      if (!seg_start_step(p.dirbit[ci.k], t, gm.L, p.kchunk)) {  // h_{-1} = 0; GSPN-local resets
        acc = tp.b * hp[r];
        if (r >= 1) acc = fmaf(tp.a, hp[r - 1], acc);
        if (r <= gm.P - 2) acc = fmaf(tp.c, hp[r + 1], acc);
      }
      const float v = fmaf(to_f(lam[off]), to_f(x[off]), acc);
      hc[r] = v;
      h[off] = from_f<T>(v);
    }
    __syncthreads();
    float* tmp = hp; hp = hc; hc = tmp;
  }
}

// Backward: adjoint recurrence in reverse step order.
// kPerChannel (G == C): the chain owns its taps, so the normalisation Jacobian is applied here;
// otherwise the normalised-tap gradients are summed over the group's channels into fp32 workspace
// and finish_dw_kernel applies the Jacobian.
template <typename T, bool kPerChannel>
__global__ void __launch_bounds__(1024) bwd_generic_kernel(ScanParams p) {
  extern __shared__ float smem[];
  const ChainIdx ci = chain_idx(p, blockIdx.x);
  const DirGeom gm = dir_geom(p.dirbit[ci.k], p.H, p.W);
  const int64_t HW = p.H * p.W;
  const T* x = static_cast<const T*>(p.x) + ci.bc * HW;
  const T* lam = static_cast<const T*>(p.lam) + ci.chain * HW;
  const T* h = static_cast<const T*>(p.h) + ci.chain * HW;
  const T* dh = static_cast<const T*>(p.dh) + ci.chain * HW;
  const int64_t wplane = (ci.k * p.B + ci.b) * p.G + ci.g;
  const T* wl = static_cast<const T*>(p.wl) + wplane * HW;
  const T* wm = static_cast<const T*>(p.wm) + wplane * HW;
  const T* wr = static_cast<const T*>(p.wr) + wplane * HW;
  T* dlam = static_cast<T*>(p.dlam) + ci.chain * HW;
  float* dx_acc = p.dx_acc + ci.bc * HW;
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  const int64_t P = gm.P;
  float* gn = smem;      // g_{t+1}
  float* gc = smem + P;  // g_t
  for (int64_t t = gm.L - 1; t >= 0; --t) {
    for (int64_t r = threadIdx.x; r < P; r += blockDim.x) {
      const int64_t off = gm.base + t * gm.ts + r * gm.rs;
      float g = to_f(dh[off]);
      if (t + 1 < gm.L && !seg_start_step(p.dirbit[ci.k], t + 1, gm.L, p.kchunk)) {
        const int64_t on = off + gm.ts;  // pixel (t+1, r)
        const Taps tm = make_taps(to_f(wl[on]), to_f(wm[on]), to_f(wr[on]), r >= 1, r <= P - 2, prenorm);
        g = fmaf(tm.b, gn[r], g);
        if (r + 1 <= P - 1) {
          const int64_t o = on + gm.rs;
          const Taps tr = make_taps(to_f(wl[o]), to_f(wm[o]), to_f(wr[o]), true, r + 1 <= P - 2, prenorm);
          g = fmaf(tr.a, gn[r + 1], g);
        }
        if (r >= 1) {
          const int64_t o = on - gm.rs;
          const Taps tl = make_taps(to_f(wl[o]), to_f(wm[o]), to_f(wr[o]), r - 1 >= 1, true, prenorm);
          g = fmaf(tl.c, gn[r - 1], g);
        }
      }
      gc[r] = g;
      dlam[off] = from_f<T>(g * to_f(x[off]));
      atomicAdd(dx_acc + off, g * to_f(lam[off]));
      float Da = 0.f, Db = 0.f, Dc = 0.f;
      const bool has_prev = !seg_start_step(p.dirbit[ci.k], t, gm.L, p.kchunk);
      if (has_prev) {
        const int64_t op = off - gm.ts;  // pixel (t-1, r)
        Db = g * to_f(h[op]);
        if (r >= 1) Da = g * to_f(h[op - gm.rs]);
        if (r <= P - 2) Dc = g * to_f(h[op + gm.rs]);
      }
      if (kPerChannel) {
        float ol, om, orr;
        jacobian(to_f(wl[off]), to_f(wm[off]), to_f(wr[off]), r >= 1, r <= P - 2, prenorm, Da, Db, Dc, ol, om, orr);
        static_cast<T*>(p.dwl)[wplane * HW + off] = from_f<T>(r >= 1 ? ol : 0.f);
        static_cast<T*>(p.dwm)[wplane * HW + off] = from_f<T>(om);
        static_cast<T*>(p.dwr)[wplane * HW + off] = from_f<T>(r <= P - 2 ? orr : 0.f);
      } else {
        if (has_prev) {
          if (r >= 1) atomicAdd(p.dwa_l + wplane * HW + off, Da);
          atomicAdd(p.dwa_m + wplane * HW + off, Db);
          if (r <= P - 2) atomicAdd(p.dwa_r + wplane * HW + off, Dc);
        }
      }
    }
    __syncthreads();
    float* tmp = gn; gn = gc; gc = tmp;
  }
}

template <typename T>
__global__ void finish_dx_kernel(const float* __restrict__ acc, T* __restrict__ dx, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dx[i] = from_f<T>(acc[i]);
}

// dw = Jacobian of the row normalisation applied to the group-summed tap gradients:
// q = a Da + b Db + c Dc; dw_l = [r>=1](Da - q)/S, dw_m = (Db - q)/S, dw_r = [r<=P-2](Dc - q)/S.
template <typename T>
__global__ void finish_dw_kernel(ScanParams p) {
  const int64_t HW = p.H * p.W;
  const int64_t n = p.D * p.B * p.G * HW;
  const bool prenorm = p.flags & GSPN_FLAG_PRENORMALIZED;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / (p.B * p.G * HW));
    const int64_t off = e % HW;
    const int64_t i = off / p.W, j = off % p.W;
    const bool vert = is_vertical(p.dirbit[k]);
    const int64_t r = vert ? j : i;
    const int64_t P = vert ? p.W : p.H;
    const bool hl = r >= 1, hr = r <= P - 2;
    const float Da = p.dwa_l[e], Db = p.dwa_m[e], Dc = p.dwa_r[e];
    float ol, om, orr;
    jacobian(to_f(static_cast<const T*>(p.wl)[e]), to_f(static_cast<const T*>(p.wm)[e]),
             to_f(static_cast<const T*>(p.wr)[e]), hl, hr, prenorm, Da, Db, Dc, ol, om, orr);
    if (p.flags & GSPN_FLAG_DW_F32) {  // fp32 partial sums (cross-device reduction)
      static_cast<float*>(p.dwl)[e] = hl ? ol : 0.f;
      static_cast<float*>(p.dwm)[e] = om;
      static_cast<float*>(p.dwr)[e] = hr ? orr : 0.f;
    } else {
      static_cast<T*>(p.dwl)[e] = from_f<T>(hl ? ol : 0.f);
      static_cast<T*>(p.dwm)[e] = from_f<T>(om);
      static_cast<T*>(p.dwr)[e] = from_f<T>(hr ? orr : 0.f);
    }
  }
}

int generic_threads(int64_t P) {
  int64_t t = (P + 31) / 32 * 32;
  if (t > 1024) t = 1024;
  if (t < 32) t = 32;
  return (int)t;
}

int grid_stride_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > int64_t{16} * device_sm_count()) b = int64_t{16} * device_sm_count();
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

int64_t generic_max_P() { return 24 * 1024; }

cudaError_t launch_fwd_generic(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches) {
  const int64_t P = p.H > p.W ? p.H : p.W;
  const size_t smem = 2 * (size_t)P * sizeof(float);
  const int64_t chains = p.D * p.B * p.C;
  const int threads = generic_threads(P);
  cudaError_t e;
  if (dt == GSPN_BF16) {
    e = cudaFuncSetAttribute(fwd_generic_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fwd_generic_kernel<__nv_bfloat16><<<(unsigned)chains, threads, smem, s>>>(p);
  } else {
    e = cudaFuncSetAttribute(fwd_generic_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fwd_generic_kernel<float><<<(unsigned)chains, threads, smem, s>>>(p);
  }
  *launches += 1;
  return cudaGetLastError();
}

template <typename T>
static cudaError_t bwd_generic_t(const ScanParams& p, cudaStream_t s, int* launches) {
  const int64_t P = p.H > p.W ? p.H : p.W;
  const size_t smem = 2 * (size_t)P * sizeof(float);
  const int64_t chains = p.D * p.B * p.C;
  const int threads = generic_threads(P);
  const bool per_channel = (p.G == p.C);
  cudaError_t e;
  if (per_channel) {
    e = cudaFuncSetAttribute(bwd_generic_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    bwd_generic_kernel<T, true><<<(unsigned)chains, threads, smem, s>>>(p);
  } else {
    e = cudaFuncSetAttribute(bwd_generic_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    bwd_generic_kernel<T, false><<<(unsigned)chains, threads, smem, s>>>(p);
  }
  *launches += 1;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int64_t n = p.B * p.C * p.H * p.W;
  finish_dx_kernel<T><<<grid_stride_blocks(n), 256, 0, s>>>(p.dx_acc, static_cast<T*>(p.dx), n);
  *launches += 1;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (!per_channel) {
    finish_dw_kernel<T><<<grid_stride_blocks(p.D * p.B * p.G * p.H * p.W), 256, 0, s>>>(p);
    *launches += 1;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_finish_dw(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches) {
  const unsigned blocks = grid_stride_blocks(p.D * p.B * p.G * p.H * p.W);
  if (dt == GSPN_BF16) finish_dw_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(p);
  else finish_dw_kernel<float><<<blocks, 256, 0, s>>>(p);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_bwd_generic(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches) {
  return dt == GSPN_BF16 ? bwd_generic_t<__nv_bfloat16>(p, s, launches) : bwd_generic_t<float>(p, s, launches);
}

}  // namespace gspn
