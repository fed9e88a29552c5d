// gspn_merge.cu — output gate and direction merge:
//   y = s * sum_d u_d (.) h_d                      (§3.2 Eq. 2, y = u (.) h per pass; the
//                                                  four passes combined; Sum or Mean, s = 1/D,
//                                                  SPEC.md:203, 263; R7)
//   dh_d = s * u_d (.) dy,  du_d = s * h_d (.) dy   (its adjoint: y is bilinear in (u, h))
//
// Pure streaming: per output element the forward reads 2D values and writes one, the backward reads
// 2D + 1 and writes 2D, with no reuse -- HBM-bound, no shared memory needed. Each thread moves whole
// 16-byte vectors (8 bf16 / 4 fp32) of every direction slab with L1-bypassing loads and streaming
// stores; the grid is a multiple of the SM count (grid-stride loop) with enough 16-byte loads in
// flight per SM (2D per vector, 2048 threads) to cover DRAM latency. fp32 arithmetic, outputs RNE.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gspn_internal.h"

namespace gspn {
namespace {

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// 16-byte vector <-> V floats.
template <typename T> struct Vec;
template <> struct Vec<__nv_bfloat16> {
  static constexpr int V = 8;
  __device__ __forceinline__ static void unpack(const uint4& q, float (&f)[V]) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  __device__ __forceinline__ static uint4 pack(const float (&f)[V]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
      w[i] = *reinterpret_cast<const uint32_t*>(&b);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <> struct Vec<float> {
  static constexpr int V = 4;
  __device__ __forceinline__ static void unpack(const uint4& q, float (&f)[V]) {
    f[0] = __uint_as_float(q.x); f[1] = __uint_as_float(q.y);
    f[2] = __uint_as_float(q.z); f[3] = __uint_as_float(q.w);
  }
  __device__ __forceinline__ static uint4 pack(const float (&f)[V]) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  }
};

// Vector kernels (N % V == 0, so every direction slab starts 16-byte aligned). nv = N / V vectors.
template <typename T, int D>
__global__ void __launch_bounds__(256) merge_fwd_vec(const T* __restrict__ h, const T* __restrict__ u,
                                                     T* __restrict__ y, int64_t N, int64_t nv, float s) {
  constexpr int V = Vec<T>::V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 hq[D], uq[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {  // all 2D loads issued before any arithmetic
      hq[d] = ld_stream(h + d * N + i * V);
      uq[d] = ld_stream(u + d * N + i * V);
    }
    float acc[V];
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] = 0.f;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      float hf[V], uf[V];
      Vec<T>::unpack(hq[d], hf);
      Vec<T>::unpack(uq[d], uf);
#pragma unroll
      for (int e = 0; e < V; ++e) acc[e] = fmaf(uf[e], hf[e], acc[e]);
    }
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] *= s;
    st_stream(y + i * V, Vec<T>::pack(acc));
  }
}

template <typename T, int D>
__global__ void __launch_bounds__(256) merge_bwd_vec(const T* __restrict__ h, const T* __restrict__ u,
                                                     const T* __restrict__ dy, T* __restrict__ dh,
                                                     T* __restrict__ du, int64_t N, int64_t nv, float s) {
  constexpr int V = Vec<T>::V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 hq[D], uq[D];
    const uint4 gq = ld_stream(dy + i * V);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      hq[d] = ld_stream(h + d * N + i * V);
      uq[d] = ld_stream(u + d * N + i * V);
    }
    float g[V];
    Vec<T>::unpack(gq, g);
#pragma unroll
    for (int e = 0; e < V; ++e) g[e] *= s;  // s * dy (s = 1 exactly for Sum)
#pragma unroll
    for (int d = 0; d < D; ++d) {
      float hf[V], uf[V], a[V], b[V];
      Vec<T>::unpack(hq[d], hf);
      Vec<T>::unpack(uq[d], uf);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        a[e] = uf[e] * g[e];
        b[e] = hf[e] * g[e];
      }
      st_stream(dh + d * N + i * V, Vec<T>::pack(a));
      st_stream(du + d * N + i * V, Vec<T>::pack(b));
    }
  }
}

// Scalar kernels for N % V != 0 (direction slabs not 16-byte aligned).
template <typename T>
__global__ void __launch_bounds__(256) merge_fwd_scalar(const T* __restrict__ h, const T* __restrict__ u,
                                                        T* __restrict__ y, int64_t N, int D, float s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int d = 0; d < D; ++d) acc = fmaf(to_f(u[d * N + i]), to_f(h[d * N + i]), acc);
    y[i] = from_f<T>(acc * s);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) merge_bwd_scalar(const T* __restrict__ h, const T* __restrict__ u,
                                                        const T* __restrict__ dy, T* __restrict__ dh,
                                                        T* __restrict__ du, int64_t N, int D, float s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const float g = to_f(dy[i]) * s;
    for (int d = 0; d < D; ++d) {
      dh[d * N + i] = from_f<T>(to_f(u[d * N + i]) * g);
      du[d * N + i] = from_f<T>(to_f(h[d * N + i]) * g);
    }
  }
}

int grid_for(int64_t work) {
  const int sms = device_sm_count();
  const int64_t full = (work + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;  // 8 x 256 threads resident per SM
  return static_cast<int>(full < cap ? (full < 1 ? 1 : full) : cap);
}

template <typename T>
cudaError_t merge_fwd_t(const void* h, const void* u, void* y, int64_t N, int D, float s, cudaStream_t st) {
  constexpr int V = Vec<T>::V;
  const T *hp = static_cast<const T*>(h), *up = static_cast<const T*>(u);
  T* yp = static_cast<T*>(y);
  if (N % V == 0) {
    const int64_t nv = N / V;
    const int g = grid_for(nv);
    switch (D) {
      case 1: merge_fwd_vec<T, 1><<<g, 256, 0, st>>>(hp, up, yp, N, nv, s); break;
      case 2: merge_fwd_vec<T, 2><<<g, 256, 0, st>>>(hp, up, yp, N, nv, s); break;
      case 3: merge_fwd_vec<T, 3><<<g, 256, 0, st>>>(hp, up, yp, N, nv, s); break;
      default: merge_fwd_vec<T, 4><<<g, 256, 0, st>>>(hp, up, yp, N, nv, s); break;
    }
  } else {
    merge_fwd_scalar<T><<<grid_for(N), 256, 0, st>>>(hp, up, yp, N, D, s);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t merge_bwd_t(const void* h, const void* u, const void* dy, void* dh, void* du, int64_t N, int D, float s,
                        cudaStream_t st) {
  constexpr int V = Vec<T>::V;
  const T *hp = static_cast<const T*>(h), *up = static_cast<const T*>(u), *gp = static_cast<const T*>(dy);
  T *dhp = static_cast<T*>(dh), *dup = static_cast<T*>(du);
  if (N % V == 0) {
    const int64_t nv = N / V;
    const int g = grid_for(nv);
    switch (D) {
      case 1: merge_bwd_vec<T, 1><<<g, 256, 0, st>>>(hp, up, gp, dhp, dup, N, nv, s); break;
      case 2: merge_bwd_vec<T, 2><<<g, 256, 0, st>>>(hp, up, gp, dhp, dup, N, nv, s); break;
      case 3: merge_bwd_vec<T, 3><<<g, 256, 0, st>>>(hp, up, gp, dhp, dup, N, nv, s); break;
      default: merge_bwd_vec<T, 4><<<g, 256, 0, st>>>(hp, up, gp, dhp, dup, N, nv, s); break;
    }
  } else {
    merge_bwd_scalar<T><<<grid_for(N), 256, 0, st>>>(hp, up, gp, dhp, dup, N, D, s);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_merge_fwd(const void* h, const void* u, void* y, int64_t N, int D, bool mean, gspn_dtype_t dt,
                             cudaStream_t st) {
  const float s = mean ? 1.f / static_cast<float>(D) : 1.f;
  return dt == GSPN_BF16 ? merge_fwd_t<__nv_bfloat16>(h, u, y, N, D, s, st) : merge_fwd_t<float>(h, u, y, N, D, s, st);
}

cudaError_t launch_merge_bwd(const void* h, const void* u, const void* dy, void* dh, void* du, int64_t N, int D,
                             bool mean, gspn_dtype_t dt, cudaStream_t st) {
  const float s = mean ? 1.f / static_cast<float>(D) : 1.f;
  return dt == GSPN_BF16 ? merge_bwd_t<__nv_bfloat16>(h, u, dy, dh, du, N, D, s, st)
                         : merge_bwd_t<float>(h, u, dy, dh, du, N, D, s, st);
}

}  // namespace gspn
