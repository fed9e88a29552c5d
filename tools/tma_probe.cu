// tma_probe.cu — micro-benchmark of TMA streaming patterns on B200 (experiments for the horizontal
// scan tiles): each CTA streams whole [H][W] bf16 planes column-chunk by column-chunk (box = chunk
// bytes wide x 256 rows, 2 boxes per chunk for H = 512) through a ring of shared-memory stages, with
// no compute. Reports time; run under `ncu --metrics dram__bytes_read.sum` for DRAM traffic.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tools/tma_probe.cu
//   ./tma_probe <chunk_bytes 16|32|64|128> <ctas> <planes> <stages> <pair 0|1> <policy 0 first|1 normal|2 last>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap map, int planes, int W, int cw,
                                               int stages, int pair, int pol_code, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * cw * 512);
  const int esz = cw * 512;  // bytes per stage (512 rows)
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint64_t pol;
  if (pol_code == 0) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else if (pol_code == 1) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  const int cols = cw / 2;  // bf16 columns per chunk
  const int nch = W / cols;
  unsigned issued = 0, waited = 0;
  unsigned long long acc = 0;
  for (int pl = blockIdx.x; pl < planes; pl += gridDim.x) {
    for (int c = 0; c < nch; ++c) {
      // keep `stages` chunks in flight: wait for the oldest before reusing its slot
      if (issued - waited == (unsigned)stages) {
        const int s = waited % stages;
        const unsigned par = (waited / stages) & 1;
        asm volatile("{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(
                         su32(&full[s])),
                     "r"(par)
                     : "memory");
        acc += smem[(size_t)s * esz];
        ++waited;
      }
      const int s = issued % stages;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(esz) : "memory");
      for (int q = 0; q < 2; ++q)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(su32(smem + (size_t)s * esz + q * 256 * cw)),
            "l"((uint64_t)&map), "r"(c * cols), "r"(q * 256), "r"(pl), "r"(su32(&full[s])), "l"(pol)
            : "memory");
      ++issued;
      (void)pair;
    }
  }
  while (waited < issued) {
    const int s = waited % stages;
    const unsigned par = (waited / stages) & 1;
    asm volatile("{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(
                     su32(&full[s])),
                 "r"(par)
                 : "memory");
    ++waited;
  }
  sink[blockIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int cw = argc > 1 ? atoi(argv[1]) : 16;
  const int ctas = argc > 2 ? atoi(argv[2]) : 148;
  const int planes = argc > 3 ? atoi(argv[3]) : 2560;
  const int stages = argc > 4 ? atoi(argv[4]) : 4;
  const int pair = argc > 5 ? atoi(argv[5]) : 0;
  const int polc = argc > 6 ? atoi(argv[6]) : 1;
  const int H = 512, W = 512;
  void* buf;
  const size_t bytes = (size_t)planes * H * W * 2;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, ctas * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)planes};
  cuuint64_t str[2] = {(cuuint64_t)W * 2, (cuuint64_t)W * H * 2};
  cuuint32_t box[3] = {(cuuint32_t)(cw / 2), 256, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  const size_t smem = (size_t)stages * cw * 512 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<<<ctas, 64, smem>>>(map, planes, W, cw, stages, pair, polc, sink);
  cudaEventRecord(e0);
  probe<<<ctas, 64, smem>>>(map, planes, W, cw, stages, pair, polc, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("chunk %d B, ctas %d, planes %d, stages %d, policy %d: %.3f ms, %.1f GB/s (useful)\n", cw, ctas, planes, stages,
         polc, ms, bytes / (ms * 1e-3) / 1e9);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
