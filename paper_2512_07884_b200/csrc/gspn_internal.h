// gspn_internal.h — host-side interfaces between the C-ABI front end and the kernel launchers.
#pragma once

#include <cuda_runtime.h>

#include "gspn_common.cuh"

namespace gspn {

// Attributes of the current device, cached per device (gspn_device.cu).
int device_sm_count();
int device_smem_optin();

int64_t generic_max_P();
cudaError_t launch_fwd_generic(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches);
cudaError_t launch_bwd_generic(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches);

// Group-summed tap gradients (fp32 workspace dwa_*) -> dw through the normalisation Jacobian (G < C).
cudaError_t launch_finish_dw(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches);

// Small-plane path (gspn_small.cu): max(H, W) <= 32, whole planes in shared memory, one CTA per (b, c).
bool small_eligible(const ScanParams& p);
cudaError_t launch_fwd_small(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches);
cudaError_t launch_bwd_small(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches);
// Grouped weights (G < C) on small planes: one CTA per unit (b, g), taps normalised once per group,
// dw formed in-kernel (no workspace, one launch). small_grouped(): eligible (fits shared memory).
bool small_grouped(const ScanParams& p, gspn_dtype_t dt);
cudaError_t launch_bwd_small_grouped(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches);
// Grouped small planes on thread-block clusters (gspn_small_cl.cu): one CTA per (unit, direction), channels
// streamed through bulk-copied batch buffers; taken by the two launchers above when eligible.
bool small_cl_eligible(const ScanParams& p, gspn_dtype_t dt, bool bwd);
cudaError_t launch_fwd_small_cl(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches);
cudaError_t launch_bwd_small_cl(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches);

// Fast TMA-streaming path (gspn_stream.cu). *handled = false when the shape is not eligible.
// *path = "stream" or "stream-cluster" (P-split over a thread-block cluster)
cudaError_t launch_fwd_stream(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches, bool* handled,
                              const char** path);
// Backward: *path = "stream-fused" (recurrence + tap gradients in one pass, G = C) or "stream" (split; "stream-cluster" when P-split).
cudaError_t launch_bwd_stream(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches, bool* handled,
                              const char** path);
// Forward + output gate + direction merge in one cooperative launch (NEXT-1); *handled = false: fall back.
cudaError_t launch_fwd_merged(const ScanParams& p, gspn_dtype_t dt, const void* u, void* y, float scale,
                              cudaStream_t s, int* launches, bool* handled);
// Recompute-h backward (NEXT-3): forward checkpoints (p.ckpt) and the one-launch backward reading them.
bool ckpt_eligible(const ScanParams& p, gspn_dtype_t dt);
size_t ckpt_floats(const ScanParams& p, gspn_dtype_t dt);
bool launch_bwd_recompute(const ScanParams& p, gspn_dtype_t dt, cudaStream_t s, int* launches, cudaError_t* err);
size_t stream_bwd_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W, int64_t D, int64_t G, gspn_dtype_t dt);

// Output gate + direction merge (gspn_merge.cu). N = B*C*H*W elements per direction slab.
cudaError_t launch_merge_fwd(const void* h, const void* u, void* y, int64_t N, int D, bool mean, gspn_dtype_t dt,
                             cudaStream_t st);
cudaError_t launch_merge_bwd(const void* h, const void* u, const void* dy, void* dh, void* du, int64_t N, int D,
                             bool mean, gspn_dtype_t dt, cudaStream_t st);

// Proxy projections on tcgen05 (gspn_umma.cu): bf16, Co <= 512, H W % 8 == 0.
bool umma_mix_eligible(int64_t B, int64_t Ci, int64_t Co, int64_t HW, gspn_dtype_t dt);
cudaError_t launch_umma_mix(const void* in, const void* M, void* out, int64_t B, int64_t Ci, int64_t Co, int64_t HW,
                            bool trans, cudaStream_t s);
bool umma_wgrad_eligible(int64_t B, int64_t Ci, int64_t Co, int64_t HW, gspn_dtype_t dt);
cudaError_t launch_umma_wgrad(const void* dout, const void* in, float* dM, int64_t B, int64_t Ci, int64_t Co,
                              int64_t HW, cudaStream_t s);

// Proxy projections (gspn_proxy.cu).
size_t proxy_mix_smem(int64_t Ci, int64_t Co);
size_t proxy_wgrad_smem(int64_t Ci, int64_t Co);
cudaError_t launch_proxy_mix(const void* in, const void* M, void* out, int64_t B, int64_t Ci, int64_t Co, int64_t HW,
                             bool trans, gspn_dtype_t dt, cudaStream_t s);
cudaError_t launch_proxy_wgrad(const void* dout, const void* in, float* dM, int64_t B, int64_t Ci, int64_t Co,
                               int64_t HW, gspn_dtype_t dt, cudaStream_t s);

}  // namespace gspn
