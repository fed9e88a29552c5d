// Device twin of synth/__init__.py: counter-based uniform generator, bit-identical to the host one.
// Holds no arithmetic of the GSPN method (it is input generation only).
//   key = splitmix64((seed << 8) | stream); u = (splitmix64(key ^ gidx) >> 40) * 2^-24
//   v = lo + (hi - lo) * u  in fp64 with explicit RN mul/add (no FMA) -> fp32 RN -> bf16 RN
//   gidx = index_base + (i / inner) * outer_stride + (i % inner)   (shards regenerate their slice)
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int kBF16>
__global__ void fill_kernel(void* __restrict__ out, int64_t n, int64_t index_base, int64_t inner,
                            int64_t outer_stride, uint64_t key, double lo, double span) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    const uint64_t gidx = (uint64_t)(index_base + (i / inner) * outer_stride + (i % inner));
    const uint64_t bits = splitmix64(key ^ gidx) >> 40;
    const double u = (double)bits * (1.0 / 16777216.0);
    const double v = __dadd_rn(lo, __dmul_rn(span, u));
    const float f = __double2float_rn(v);
    if (kBF16) {
      static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(f);
    } else {
      static_cast<float*>(out)[i] = f;
    }
  }
}

}  // namespace

extern "C" {

// dtype: 0 = fp32, 1 = bf16. inner <= 0 means identity mapping (gidx = index_base + i).
// Returns 0 on success, 1 on bad arguments, 3 on a CUDA error.
int synth_fill(void* out, int64_t n, int64_t index_base, int64_t inner, int64_t outer_stride, uint64_t seed,
               uint32_t stream_id, double lo, double hi, int dtype, void* cuda_stream) {
  if (n < 0 || (n > 0 && out == nullptr) || (dtype != 0 && dtype != 1)) return 1;
  if (n == 0) return 0;
  if (inner <= 0) {
    inner = n;
    outer_stride = 0;
  }
  const uint64_t key = splitmix64((seed << 8) | (uint64_t)stream_id);
  const int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  if (dtype == 1)
    fill_kernel<1><<<(unsigned)blocks, threads, 0, s>>>(out, n, index_base, inner, outer_stride, key, lo, hi - lo);
  else
    fill_kernel<0><<<(unsigned)blocks, threads, 0, s>>>(out, n, index_base, inner, outer_stride, key, lo, hi - lo);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // extern "C"
