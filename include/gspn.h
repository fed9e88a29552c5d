/*
 * gspn.h — C ABI of the B200-native GSPN / GSPN-2 line-scan propagation (arxiv 2512.07884).
 *
 * Operation (§3.2 Eq. 1; §4.2 Eq. 3; §3.2):
 *   In scan coordinates (step t = 0..L-1, position r = 0..P-1) of one direction, one batch b and one
 *   channel c in weight group g = c / (C/G):
 *
 *     h_t[r] = a_t[r] h_{t-1}[r-1] + b_t[r] h_{t-1}[r] + c_t[r] h_{t-1}[r+1] + lam_t[r] x_t[r],  h_{-1} = 0
 *
 *   (a, b, c) are the row-normalised ("row-stochastic") tridiagonal taps of the raw
 *   per-pixel taps (w_l, w_m, w_r):  S = w_m + [r>=1] w_l + [r<=P-2] w_r,
 *   a = [r>=1] w_l / S,  b = w_m / S,  c = [r<=P-2] w_r / S   (out-of-range taps are dropped and the
 *   row renormalised over the in-range ones; readings R1, R2). h_{-1} = 0 follows from
 *   Eq. 4's first block row Lambda_1. With GSPN_FLAG_PRENORMALIZED the taps are used
 *   as given (still dropped out of range) and no division happens.
 *
 *   Directions ("four complementary directional passes"); canonical pixel (i, j):
 *     T2B: t = i,       r = j   (L = H, P = W)       B2T: t = H-1-i, r = j   (L = H, P = W)
 *     L2R: t = j,       r = i   (L = W, P = H)       R2L: t = W-1-j, r = i   (L = W, P = H)
 *   w_l always multiplies the neighbour with the smaller canonical parallel index (R4).
 *   The taps stored at pixel (i, j) are the row of the step matrix that produces pixel (i, j) (R5).
 *
 * Layout (all tensors dense, contiguous, row-major, element type = dtype):
 *   x                 [B, C, H, W]        shared by all directions (R6)
 *   w_l, w_m, w_r     [D, B, G, H, W]     one tap triple per pixel per group (G = C: per-channel
 *                                          weights, Eq. 1; G = 1: channel-shared weights, Eq. 3)
 *   lam, h, dh, dlam  [D, B, C, H, W]
 *   dx                [B, C, H, W]        sum over the D directions
 *   dw_l, dw_m, dw_r  [D, B, G, H, W]     gradient w.r.t. the RAW taps, summed over the group's channels
 *   D = popcount(dirs); direction slabs appear in bit order T2B, B2T, L2R, R2L.
 *
 * Ownership: every tensor pointer is a caller-owned DEVICE pointer (cudaMalloc / torch). The library
 *   allocates nothing, keeps no pointer after return, and writes only the listed outputs (and the
 *   caller's workspace). Outputs are fully overwritten, never accumulated into.
 * Execution: stream-ordered and asynchronous on `stream`; no host synchronisation inside. Device-side
 *   faults surface at the caller's next synchronisation (CUDA convention).
 * Errors: arguments are validated on the host BEFORE any CUDA call; on failure nothing is launched
 *   or written and the call returns GSPN_ERR_INVALID_ARG (detail in gspn_last_error_detail()).
 *   No C++ exception crosses this boundary.
 * Preconditions not checked on the device: taps >= 0 with S > 0 at every position, inputs finite.
 */
#ifndef GSPN_H_
#define GSPN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GSPN_OK = 0,
  GSPN_ERR_INVALID_ARG = 1, /* bad pointer / dim / flag / dtype / alignment / aliasing */
  GSPN_ERR_UNSUPPORTED = 2, /* shape the kernels cannot tile (never for BASELINE.json's configs) */
  GSPN_ERR_CUDA = 3,        /* a CUDA runtime / driver call or launch failed */
  GSPN_ERR_INTERNAL = 4     /* anything else (caught exception) */
} gspn_status_t;

typedef enum { GSPN_F32 = 0, GSPN_BF16 = 1 } gspn_dtype_t;

#define GSPN_DIR_T2B 0x1u /* step = row i ascending,     position = column j */
#define GSPN_DIR_B2T 0x2u /* step = row i descending,    position = column j */
#define GSPN_DIR_L2R 0x4u /* step = column j ascending,  position = row i    */
#define GSPN_DIR_R2L 0x8u /* step = column j descending, position = row i    */
#define GSPN_DIR_ALL 0xFu

#define GSPN_FLAG_PRENORMALIZED 0x1u /* taps already row-normalised: no division (out-of-range taps still dropped) */
#define GSPN_FLAG_FORCE_GENERIC 0x2u /* testing: force the generic (non-TMA) kernels */
#define GSPN_FLAG_MERGE_MEAN 0x4u    /* gspn_merge_*: combine the directions by Mean instead of Sum */
#define GSPN_FLAG_DW_F32 0x20u       /* gspn_bwd: dw_l/dw_m/dw_r are fp32 tensors whatever dtype (partial group sums
                                       to be reduced across devices in fp32); groups < C only,
                                       GSPN_ERR_UNSUPPORTED for groups == C */
#define GSPN_FLAG_FORCE_SPLIT 0x10u  /* testing: split every chain over a 2+-CTA cluster (P-split) even when one
                                       CTA could hold it; results must be bitwise those of the unsplit scan */

/* cudaStream_t without including CUDA headers (ABI-identical: an opaque pointer). */
typedef struct CUstream_st* gspn_stream_t;

/*
 * Forward scan, all requested directions in one persistent launch.
 *   x [B,C,H,W]; w_l/w_m/w_r [D,B,G,H,W]; lam [D,B,C,H,W]  -> h [D,B,C,H,W]
 *   B, C, H, W, groups >= 1; C % groups == 0; dirs in [1, 15]; flags subset of GSPN_FLAG_*.
 *   Every pointer non-null and 16-byte aligned; h must not overlap any input.
 */
gspn_status_t gspn_fwd(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                       void* h, int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                       gspn_dtype_t dtype, uint32_t flags, gspn_stream_t stream);

/*
 * Backward (adjoint, reverse-order) scan given the saved forward output h and the upstream gradient dh.
 *   Produces dx [B,C,H,W] (summed over directions), dlam [D,B,C,H,W] and dw_l/dw_m/dw_r [D,B,G,H,W]
 *   (gradient w.r.t. the raw taps, chained through the row normalisation and summed over the group's
 *   channels; zero for out-of-range taps and for every tap at step t = 0, whose h_{-1} = 0).
 *   workspace: caller-owned device scratch of at least gspn_bwd_workspace_bytes(...) bytes (16-byte
 *   aligned; may be NULL when that size is 0). Its contents on entry are ignored; the library
 *   initialises it on `stream`. No output may overlap any input, another output or the workspace.
 * Determinism: gspn_fwd is bitwise deterministic and independent of the tiling (P-split clusters, chain
 *   packing). gspn_bwd sums dx over the directions and dw over a group's channels in a fixed order on the
 *   streaming and grouped small-plane paths (bitwise run-to-run); the generic kernels
 *   (GSPN_FLAG_FORCE_GENERIC, or shapes no fast path tiles) and the per-plane small kernels used for
 *   groups < C when the grouped kernel does not fit shared memory add with fp32 atomics, so their
 *   dx / dw may differ in the last bits between runs.
 */
gspn_status_t gspn_bwd(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                       const void* h, const void* dh, void* dx, void* dw_l, void* dw_m, void* dw_r, void* dlam,
                       int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                       gspn_dtype_t dtype, uint32_t flags, void* workspace, size_t workspace_bytes,
                       gspn_stream_t stream);

/*
 * GSPN-local variant (§3.2: "splits each row or column into fixed-length segments of size
 * kchunk and confines propagation to within those segments"). The scan axis of
 * every direction is cut into segments of kchunk steps fixed on the canonical image grid (canonical
 * row i for T2B/B2T, column j for L2R/R2L, in segment i / kchunk resp. j / kchunk; the last segment may
 * be short), and h restarts from 0 at each segment's first step in scan order (
 * DESIGN.md R19). kchunk = 0 (or >= the scan length) is the global scan: gspn_fwd / gspn_bwd are
 * exactly these calls with kchunk = 0. kchunk < 0 is GSPN_ERR_INVALID_ARG. In the backward, the taps of a
 * segment's first step get dw = 0. Everything else as gspn_fwd / gspn_bwd (same workspace size).
 */
gspn_status_t gspn_fwd_local(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                             void* h, int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                             int64_t kchunk, gspn_dtype_t dtype, uint32_t flags, gspn_stream_t stream);
gspn_status_t gspn_bwd_local(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                             const void* h, const void* dh, void* dx, void* dw_l, void* dw_m, void* dw_r, void* dlam,
                             int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                             int64_t kchunk, gspn_dtype_t dtype, uint32_t flags, void* workspace,
                             size_t workspace_bytes, gspn_stream_t stream);

/* Workspace bytes gspn_bwd needs for this problem (0 on invalid arguments). */
size_t gspn_bwd_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                                gspn_dtype_t dtype);

/* Algorithmic HBM bytes of one call (each input read once, each output written once):
 *   fwd = s * (N (1 + 2D) + 3 D N_w),  bwd = 2 * fwd,  N = B C H W,  N_w = B G H W. */
double gspn_algorithmic_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                              gspn_dtype_t dtype, int backward);

/*
 * Output gate + direction merge. PAPER.md:84-88 (§3.2, Eq. 2) gates each
 * pass's state, y = u (.) h; the four directional passes are "combined" -- by Sum, or by
 * Mean with GSPN_FLAG_MERGE_MEAN (R7):
 *     y = s * sum_d u_d (.) h_d,      s = 1 (Sum) or 1/D (Mean)
 *   h, u [D,B,C,H,W] (slabs in bit order, as gspn_fwd's h)  ->  y [B,C,H,W]
 * Arithmetic in fp32, y rounded once to dtype. flags: 0 or GSPN_FLAG_MERGE_MEAN. Pointers non-null,
 * 16-byte aligned; y must not overlap h or u. One launch; HBM-bound (s N (2D + 1) bytes).
 */
gspn_status_t gspn_merge_fwd(const void* h, const void* u, void* y, int64_t B, int64_t C, int64_t H, int64_t W,
                             uint32_t dirs, gspn_dtype_t dtype, uint32_t flags, gspn_stream_t stream);

/*
 * Adjoint of gspn_merge_fwd given dy [B,C,H,W]:  dh_d = s * u_d (.) dy,  du_d = s * h_d (.) dy
 * (dh, du [D,B,C,H,W]; dh is what gspn_bwd takes as its upstream gradient). No output may overlap an
 * input or the other output. One launch; s N (4D + 1) bytes.
 */
gspn_status_t gspn_merge_bwd(const void* h, const void* u, const void* dy, void* dh, void* du, int64_t B, int64_t C,
                             int64_t H, int64_t W, uint32_t dirs, gspn_dtype_t dtype, uint32_t flags,
                             gspn_stream_t stream);

/*
 * Forward scan AND output gate + direction merge in one call (PAPER.md:84-89
 * Eq. 2): y = s sum_d u_d (.) h_d [B,C,H,W] with u [D,B,C,H,W] (s = 1, or 1/D with GSPN_FLAG_MERGE_MEAN).
 * h [D,B,C,H,W] is also written when non-NULL (training keeps it for gspn_bwd_merged); with h = NULL it
 * lives in the workspace (>= gspn_fwd_merged_workspace_bytes(...) bytes; may be NULL when h is given).
 * Unpacked / packed chains without P-split: one cooperative launch (scan | grid barrier | merge;
 * gspn_last_path() "stream-merged"); otherwise gspn_fwd then gspn_merge_fwd ("merged-unfused").
 * flags: GSPN_FLAG_PRENORMALIZED, GSPN_FLAG_MERGE_MEAN, GSPN_FLAG_FORCE_GENERIC.
 */
gspn_status_t gspn_fwd_merged(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                              const void* u, void* h, void* y, int64_t B, int64_t C, int64_t H, int64_t W,
                              uint32_t dirs, int64_t groups, gspn_dtype_t dtype, uint32_t flags, void* workspace,
                              size_t workspace_bytes, gspn_stream_t stream);
size_t gspn_fwd_merged_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                                       gspn_dtype_t dtype);

/*
 * Backward through the scan AND the output gate + direction merge in one call (SURVEY.md §8(f) NEXT-1,
 * PAPER.md:84-88 Eq. 2): given the merge's upstream gradient dy [B,C,H,W] and the gate u [D,B,C,H,W],
 * the scan's upstream gradient is dh_d = s u_d (.) dy (s = 1, or 1/D with GSPN_FLAG_MERGE_MEAN) and the
 * gate's gradient du_d = s h_d (.) dy [D,B,C,H,W] is written alongside dx, dw, dlam (gspn_bwd's outputs).
 * On the fused path (per-channel weights, unpacked or packed, not P-split) dh is formed inside the single
 * backward launch and never stored (gspn_last_path() "stream-fused-merged"); otherwise the merge adjoint
 * writes dh into the workspace and gspn_bwd follows ("merged-unfused"). flags: GSPN_FLAG_PRENORMALIZED,
 * GSPN_FLAG_MERGE_MEAN, GSPN_FLAG_FORCE_GENERIC. workspace: >= gspn_bwd_merged_workspace_bytes(...).
 * Other conventions as gspn_bwd.
 */
gspn_status_t gspn_bwd_merged(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                              const void* h, const void* u, const void* dy, void* dx, void* dw_l, void* dw_m,
                              void* dw_r, void* dlam, void* du, int64_t B, int64_t C, int64_t H, int64_t W,
                              uint32_t dirs, int64_t groups, gspn_dtype_t dtype, uint32_t flags, void* workspace,
                              size_t workspace_bytes, gspn_stream_t stream);
size_t gspn_bwd_merged_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                                       gspn_dtype_t dtype);

/*
 * Recompute-h backward (activation checkpointing inside the kernels).
 * gspn_fwd_ckpt is gspn_fwd that also writes fp32 checkpoints of h -- one row per half-tile of KS = 16/s
 * steps (s = element size), per chain -- into `ckpt` (gspn_ckpt_bytes(...) bytes, contents implementation-
 * defined) and may skip h itself (h = NULL: the forward then writes s (1 + 2D) N + ... bytes less).
 * gspn_bwd_recompute is gspn_bwd without h: each half-tile's h is recomputed in registers from the
 * checkpoint (Eq. 1, fp32: the tap gradients see h unrounded), the tap gradients of every direction are
 * formed inside the adjoint recurrence, and one output phase forms dlam and dx -- one cooperative launch
 * (gspn_last_path() "stream-recompute"). Shapes without checkpoints (grouped weights, packed small planes,
 * P-split chains, H or W not a multiple of 32/s) keep nothing in the forward ("ckpt-deferred") and the
 * backward re-runs the forward into its workspace ("recompute-unfused"). flags: GSPN_FLAG_PRENORMALIZED,
 * GSPN_FLAG_FORCE_GENERIC. workspace: >= gspn_bwd_recompute_workspace_bytes(...). Otherwise as gspn_fwd /
 * gspn_bwd.
 */
gspn_status_t gspn_fwd_ckpt(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                            void* h, float* ckpt, int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs,
                            int64_t groups, gspn_dtype_t dtype, uint32_t flags, gspn_stream_t stream);
gspn_status_t gspn_bwd_recompute(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                                 const float* ckpt, const void* dh, void* dx, void* dw_l, void* dw_m, void* dw_r,
                                 void* dlam, int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs,
                                 int64_t groups, gspn_dtype_t dtype, uint32_t flags, void* workspace,
                                 size_t workspace_bytes, gspn_stream_t stream);
size_t gspn_ckpt_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups, gspn_dtype_t dtype);
size_t gspn_bwd_recompute_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                                          gspn_dtype_t dtype);

/*
 * Compact-channel proxy projections (§4.2 "project the input tensor
 * x in R^{N x C x H x W} into a lower-dimensional proxy subspace x_proxy in R^{N x C_proxy x H x W}",
 * PAPER.md:172 "expand back to C with a learned 1x1 projection"). A 1x1 projection mixes channels at
 * every pixel:
 *     out[b, o, :] = sum_i M[o, i] in[b, i, :]      in [B, Ci, H, W] -> out [B, Co, H, W]
 *   M [Co, Ci] row-major in dtype, or, with GSPN_FLAG_PROXY_TRANSPOSE, M stored [Ci, Co] (its transpose
 *   is used): the data gradient of a projection by M is the projection of the upstream gradient by M^T.
 *   Down-projection: M = P_down [C_proxy, C]; up-projection: M = P_up [C, C_proxy]. fp32 accumulation.
 *   H*W must be even. One launch. bf16 with Co <= 512 and H*W % 8 == 0 runs on the tensor cores
 *   (tcgen05.mma, fp32 accumulator in TMEM; gspn_last_path() "proxy-umma"), anything else on SIMT FMAs
 *   ("proxy"), which needs Co*Ci <= 49152 (M staged in shared memory).
 */
#define GSPN_FLAG_PROXY_TRANSPOSE 0x8u
#define GSPN_FLAG_PROXY_SIMT 0x10u /* testing: gspn_proxy_mix on the SIMT kernel instead of tcgen05 */
gspn_status_t gspn_proxy_mix(const void* in, const void* M, void* out, int64_t B, int64_t Ci, int64_t Co, int64_t H,
                             int64_t W, gspn_dtype_t dtype, uint32_t flags, gspn_stream_t stream);
/*
 * Weight gradient of gspn_proxy_mix:  dM[o, i] = sum_{b, pixels} dout[b, o, :] . in[b, i, :]
 *   dout [B, Co, H, W], in [B, Ci, H, W] (dtype) -> dM [Co, Ci] in FP32 (overwritten; a reduction over
 *   B H W terms). SIMT path: (Co + Ci) * 33 + Co * Ci <= 49152. A memset and one launch (fp32 atomics across CTAs,
 *   so the summation order -- not the result beyond fp32 rounding -- varies between runs). bf16 with
 *   Co, Ci <= 512 and H*W % 8 == 0 runs on the tensor cores (each CTA's share of the pixels accumulated in
 *   TMEM; gspn_last_path() "proxy-umma").
 */
gspn_status_t gspn_proxy_wgrad(const void* dout, const void* in, float* dM, int64_t B, int64_t Ci, int64_t Co,
                               int64_t H, int64_t W, gspn_dtype_t dtype, gspn_stream_t stream);

const char* gspn_status_string(gspn_status_t s);
/* Thread-local detail string of the last failing call on this thread (names the offending argument). */
const char* gspn_last_error_detail(void);
/* Name of the kernel path the last successful call on this thread launched ("generic", "stream", ...). */
const char* gspn_last_path(void);
/* Number of kernel launches the last successful call on this thread issued (memsets excluded). */
int gspn_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* GSPN_H_ */
