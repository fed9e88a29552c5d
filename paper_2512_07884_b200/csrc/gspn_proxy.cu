// gspn_proxy.cu — compact-channel proxy projections: the 1x1 projections that
// take x [B, C, H, W] into the proxy space the scan runs in, and back (§4.2 "project the
// input tensor ... into a lower-dimensional proxy subspace x_proxy in R^{N x C_proxy x H x W}";
// PAPER.md:172 "expand back to C with a learned 1x1 projection"):
//   mix:    out[b, o, n] = sum_i M[o, i] in[b, i, n]        (n over H W; M [Co, Ci], or M^T when stored [Ci, Co])
//   wgrad:  dM[o, i]     = sum_{b, n} dout[b, o, n] in[b, i, n]
// Down-projection: M = P_down [C_proxy, C]; up: M = P_up [C, C_proxy]; their data gradients are the same
// mix with M^T, their weight gradients `wgrad`.
//
// Roofline: with C_proxy << C (8 of 384 at BASELINE configs[2], 40 of 320 at configs[4]) a pixel's mix
// costs 2 C C_proxy flops for (C + C_proxy) s bytes: ~8 flop/byte in bf16 at C_proxy = 8, far below the
// tensor-core ridge (~300 flop/byte on B200) -- HBM-bound, so SIMT FMAs at streaming speed are the
// roofline-correct choice and tcgen05 would only pay for C_proxy in the hundreds.
// mix: one thread per (b, 8-output block, pixel pair); M staged in shared memory (fp32), broadcast reads;
// consecutive threads take consecutive pixel pairs (coalesced 4- / 8-byte loads and stores).
// wgrad: one CTA per pixel range; the range is staged through shared memory in 32-pixel tiles (fp32),
// each thread owns (o, i) pairs and keeps their partial sums in a shared accumulator; one fp32 atomic
// add per pair and CTA into the caller's fp32 dM.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gspn_common.cuh"
#include "gspn_internal.h"

namespace gspn {
namespace {

constexpr int kOB = 8;  // outputs per thread in mix

template <typename T> struct Pair;  // two consecutive elements
template <> struct Pair<__nv_bfloat16> {
  __device__ __forceinline__ static void ld(const __nv_bfloat16* p, float& a, float& b) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
    a = __uint_as_float(u << 16);
    b = __uint_as_float(u & 0xFFFF0000u);
  }
  __device__ __forceinline__ static void st(__nv_bfloat16* p, float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    *reinterpret_cast<__nv_bfloat162*>(p) = v;
  }
};
template <> struct Pair<float> {
  __device__ __forceinline__ static void ld(const float* p, float& a, float& b) {
    const float2 u = *reinterpret_cast<const float2*>(p);
    a = u.x; b = u.y;
  }
  __device__ __forceinline__ static void st(float* p, float a, float b) { *reinterpret_cast<float2*>(p) = make_float2(a, b); }
};

// kTrans: M stored [Ci, Co] (use its transpose). HW even (pixel pairs).
template <typename T, bool kTrans>
__global__ void __launch_bounds__(256) mix_kernel(const T* __restrict__ in, const T* __restrict__ M, T* __restrict__ out,
                                                  int B, int Ci, int Co, int HW) {
  extern __shared__ float Ms[];  // [Co][Ci] fp32
  for (int e = threadIdx.x; e < Co * Ci; e += blockDim.x) {
    const int o = e / Ci, i = e - o * Ci;
    Ms[e] = to_f(kTrans ? M[i * Co + o] : M[e]);
  }
  __syncthreads();
  const int npair = HW / 2, nob = (Co + kOB - 1) / kOB;
  const int64_t total = static_cast<int64_t>(B) * nob * npair;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int pp = static_cast<int>(t % npair);
    const int64_t r = t / npair;
    const int ob = static_cast<int>(r % nob), b = static_cast<int>(r / nob);
    const int o0 = ob * kOB;
    float acc[kOB][2];
#pragma unroll
    for (int q = 0; q < kOB; ++q) acc[q][0] = acc[q][1] = 0.f;
    const T* src = in + static_cast<int64_t>(b) * Ci * HW + 2 * pp;
#pragma unroll 4
    for (int i = 0; i < Ci; ++i) {
      float a0, a1;
      Pair<T>::ld(src + static_cast<int64_t>(i) * HW, a0, a1);
#pragma unroll
      for (int q = 0; q < kOB; ++q) {
        const float m = (o0 + q < Co) ? Ms[(o0 + q) * Ci + i] : 0.f;
        acc[q][0] = fmaf(m, a0, acc[q][0]);
        acc[q][1] = fmaf(m, a1, acc[q][1]);
      }
    }
    T* dst = out + static_cast<int64_t>(b) * Co * HW + 2 * pp;
#pragma unroll
    for (int q = 0; q < kOB; ++q)
      if (o0 + q < Co) Pair<T>::st(dst + static_cast<int64_t>(o0 + q) * HW, acc[q][0], acc[q][1]);
  }
}

// Down-projection shape (Co <= kOB, Ci >= 64): the Ci reduction is split over kKS thread slices of a
// CTA (each slice sums Ci / kKS channels for the same 32 pixel pairs), partial sums meet in shared
// memory -- 8x the threads of mix_kernel, whose per-thread Ci loop was latency-bound at 98 CTAs.
constexpr int kKS = 8;
template <typename T, bool kTrans>
__global__ void __launch_bounds__(256) mix_splitk_kernel(const T* __restrict__ in, const T* __restrict__ M,
                                                         T* __restrict__ out, int B, int Ci, int Co, int HW) {
  extern __shared__ float Ms[];  // [Co][Ci] fp32, then partials [kKS][kOB][64]
  float* part = Ms + Co * Ci;
  for (int e = threadIdx.x; e < Co * Ci; e += blockDim.x) {
    const int o = e / Ci, i = e - o * Ci;
    Ms[e] = to_f(kTrans ? M[i * Co + o] : M[e]);
  }
  const int npair = HW / 2;
  const int nblk = (npair + 31) / 32;  // 32 pixel pairs per CTA iteration
  const int ks = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cs = (Ci + kKS - 1) / kKS, i0 = ks * cs, i1 = min(Ci, i0 + cs);
  for (int64_t blk = blockIdx.x; blk < static_cast<int64_t>(B) * nblk; blk += gridDim.x) {
    const int b = static_cast<int>(blk / nblk), pb = static_cast<int>(blk % nblk);
    const int pp = pb * 32 + lane;
    float acc[kOB][2];
#pragma unroll
    for (int q = 0; q < kOB; ++q) acc[q][0] = acc[q][1] = 0.f;
    __syncthreads();  // Ms staged / previous iteration's partials consumed
    if (pp < npair) {
      const T* src = in + static_cast<int64_t>(b) * Ci * HW + 2 * pp;
#pragma unroll 4
      for (int i = i0; i < i1; ++i) {
        float a0, a1;
        Pair<T>::ld(src + static_cast<int64_t>(i) * HW, a0, a1);
#pragma unroll
        for (int q = 0; q < kOB; ++q) {
          const float m = q < Co ? Ms[q * Ci + i] : 0.f;
          acc[q][0] = fmaf(m, a0, acc[q][0]);
          acc[q][1] = fmaf(m, a1, acc[q][1]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kOB; ++q) {
      part[(ks * kOB + q) * 64 + 2 * lane] = acc[q][0];
      part[(ks * kOB + q) * 64 + 2 * lane + 1] = acc[q][1];
    }
    __syncthreads();
    // 256 threads finish kOB x 64 outputs: thread -> (q, pixel pair)
    for (int e = threadIdx.x; e < kOB * 32; e += blockDim.x) {
      const int q = e >> 5, l = e & 31, p2 = pb * 32 + l;
      if (q >= Co || p2 >= npair) continue;
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int k = 0; k < kKS; ++k) {
        s0 += part[(k * kOB + q) * 64 + 2 * l];
        s1 += part[(k * kOB + q) * 64 + 2 * l + 1];
      }
      Pair<T>::st(out + (static_cast<int64_t>(b) * Co + q) * HW + 2 * p2, s0, s1);
    }
  }
}

constexpr int kPT = 32;        // pixels per wgrad tile
constexpr int kPTS = kPT + 1;  // staged row stride: odd, so threads on consecutive channels hit distinct banks

// kSmall: 0 generic pair loop (shared accumulators); 1 Co <= 8 (down-projection weights); 2 Ci <= 8
// (up-projection weights). kSlots: large-side channels per thread (large side <= kSlots * 256).
constexpr int kSlots = 2;
template <typename T, int kSmall>
__global__ void __launch_bounds__(256) wgrad_kernel(const T* __restrict__ dout, const T* __restrict__ in,
                                                    float* __restrict__ dM, int B, int Ci, int Co, int HW,
                                                    int64_t px_per_cta) {
  extern __shared__ float sm[];
  float racc[kSlots][8];
#pragma unroll
  for (int sl = 0; sl < kSlots; ++sl)
#pragma unroll
    for (int q = 0; q < 8; ++q) racc[sl][q] = 0.f;
  float* so = sm;                       // [Co][kPTS]
  float* si = so + Co * kPTS;           // [Ci][kPTS]
  float* acc = si + Ci * kPTS;          // [Co * Ci]
  const int npairs = Co * Ci;
  for (int e = threadIdx.x; e < npairs; e += blockDim.x) acc[e] = 0.f;
  const int64_t npx = static_cast<int64_t>(B) * HW;
  const int64_t p0 = blockIdx.x * px_per_cta;
  const int64_t p1 = p0 + px_per_cta < npx ? p0 + px_per_cta : npx;
  __shared__ int64_t offo[kPT], offi[kPT];  // per tile slot: element offset of channel 0 in dout / in
  for (int64_t base = p0; base < p1; base += kPT) {
    const int n = static_cast<int>(p1 - base < kPT ? p1 - base : kPT);
    __syncthreads();
    if (threadIdx.x < kPT) {
      const int64_t gp = base + threadIdx.x;  // flat (b, pixel): one division per slot, not per element
      const int64_t b = gp / HW, px = gp - b * HW;
      offo[threadIdx.x] = b * Co * HW + px;
      offi[threadIdx.x] = b * Ci * HW + px;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < (Co + Ci) * kPT; e += blockDim.x) {
      const int ch = e >> 5, k = e & (kPT - 1);  // kPT = 32
      float v = 0.f;
      if (k < n)
        v = ch < Co ? to_f(dout[offo[k] + static_cast<int64_t>(ch) * HW])
                    : to_f(in[offi[k] + static_cast<int64_t>(ch - Co) * HW]);
      sm[ch * kPTS + k] = v;  // so and si are contiguous: channel ch of the stacked [Co + Ci][kPTS] tile
    }
    __syncthreads();
    if (kSmall == 0) {
      for (int e = threadIdx.x; e < npairs; e += blockDim.x) {
        const int o = e / Ci, i = e - o * Ci;
        const float* a = so + o * kPTS;
        const float* c = si + i * kPTS;
        float s = 0.f;
#pragma unroll 8
        for (int k = 0; k < kPT; ++k) s = fmaf(a[k], c[k], s);
        acc[e] += s;
      }
    } else {
      // register-blocked: the small side (<= 8 channels) is read as broadcasts, each thread owns up to
      // kSlots channels of the large side and all small-side partners, sums stay in registers
      const int nsm = kSmall == 1 ? Co : Ci, nlg = kSmall == 1 ? Ci : Co;
      const float* sml = kSmall == 1 ? so : si;
      const float* lrg = kSmall == 1 ? si : so;
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) {
        const int l = threadIdx.x + sl * blockDim.x;
        if (l >= nlg) break;
#pragma unroll 4
        for (int k = 0; k < kPT; ++k) {
          const float c = lrg[l * kPTS + k];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < nsm) racc[sl][q] = fmaf(sml[q * kPTS + k], c, racc[sl][q]);
        }
      }
    }
  }
  if (kSmall != 0) {
    const int nsm = kSmall == 1 ? Co : Ci, nlg = kSmall == 1 ? Ci : Co;
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) {
      const int l = threadIdx.x + sl * blockDim.x;
      if (l >= nlg) break;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < nsm) atomicAdd(dM + (kSmall == 1 ? q * Ci + l : l * Ci + q), racc[sl][q]);
    }
    return;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < npairs; e += blockDim.x) atomicAdd(dM + e, acc[e]);
}

int sms() { return device_sm_count(); }

template <typename T>
cudaError_t mix_t(const void* in, const void* M, void* out, int B, int Ci, int Co, int HW, bool trans, cudaStream_t s) {
  if (Co <= kOB && Ci >= 64) {
    const size_t smem = (static_cast<size_t>(Co) * Ci + kKS * kOB * 64) * sizeof(float);
    auto k = trans ? mix_splitk_kernel<T, true> : mix_splitk_kernel<T, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int64_t nblk = static_cast<int64_t>(B) * ((HW / 2 + 31) / 32);
    const int64_t cap = static_cast<int64_t>(sms()) * 8;
    k<<<static_cast<unsigned>(nblk < cap ? nblk : cap), 256, smem, s>>>(
        static_cast<const T*>(in), static_cast<const T*>(M), static_cast<T*>(out), B, Ci, Co, HW);
    return cudaGetLastError();
  }
  const size_t smem = static_cast<size_t>(Co) * Ci * sizeof(float);
  auto k = trans ? mix_kernel<T, true> : mix_kernel<T, false>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t total = static_cast<int64_t>(B) * ((Co + kOB - 1) / kOB) * (HW / 2);
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sms()) * 8;
  if (blocks > cap) blocks = cap;
  k<<<static_cast<unsigned>(blocks < 1 ? 1 : blocks), 256, smem, s>>>(static_cast<const T*>(in), static_cast<const T*>(M),
                                                                     static_cast<T*>(out), B, Ci, Co, HW);
  return cudaGetLastError();
}

template <typename T>
cudaError_t wgrad_t(const void* dout, const void* in, float* dM, int B, int Ci, int Co, int HW, cudaStream_t s) {
  const size_t smem = (static_cast<size_t>(Co + Ci) * kPTS + static_cast<size_t>(Co) * Ci) * sizeof(float);
  const int mode = (Co <= 8 && Ci <= kSlots * 256) ? 1 : (Ci <= 8 && Co <= kSlots * 256) ? 2 : 0;
  auto kern = mode == 1 ? wgrad_kernel<T, 1> : mode == 2 ? wgrad_kernel<T, 2> : wgrad_kernel<T, 0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(dM, 0, static_cast<size_t>(Co) * Ci * sizeof(float), s);
  if (e != cudaSuccess) return e;
  const int64_t npx = static_cast<int64_t>(B) * HW;
  int64_t ctas = sms() * 2;
  int64_t per = (npx + ctas - 1) / ctas;
  per = (per + kPT - 1) / kPT * kPT;
  ctas = (npx + per - 1) / per;
  kern<<<static_cast<unsigned>(ctas), 256, smem, s>>>(static_cast<const T*>(dout), static_cast<const T*>(in), dM, B, Ci,
                                                      Co, HW, per);
  return cudaGetLastError();
}

}  // namespace

size_t proxy_mix_smem(int64_t Ci, int64_t Co) { return static_cast<size_t>(Ci * Co + kKS * kOB * 64) * sizeof(float); }
size_t proxy_wgrad_smem(int64_t Ci, int64_t Co) {
  return (static_cast<size_t>(Co + Ci) * kPTS + static_cast<size_t>(Co * Ci)) * sizeof(float);
}

cudaError_t launch_proxy_mix(const void* in, const void* M, void* out, int64_t B, int64_t Ci, int64_t Co, int64_t HW,
                             bool trans, gspn_dtype_t dt, cudaStream_t s) {
  return dt == GSPN_BF16 ? mix_t<__nv_bfloat16>(in, M, out, (int)B, (int)Ci, (int)Co, (int)HW, trans, s)
                         : mix_t<float>(in, M, out, (int)B, (int)Ci, (int)Co, (int)HW, trans, s);
}

cudaError_t launch_proxy_wgrad(const void* dout, const void* in, float* dM, int64_t B, int64_t Ci, int64_t Co,
                               int64_t HW, gspn_dtype_t dt, cudaStream_t s) {
  return dt == GSPN_BF16 ? wgrad_t<__nv_bfloat16>(dout, in, dM, (int)B, (int)Ci, (int)Co, (int)HW, s)
                         : wgrad_t<float>(dout, in, dM, (int)B, (int)Ci, (int)Co, (int)HW, s);
}

}  // namespace gspn
