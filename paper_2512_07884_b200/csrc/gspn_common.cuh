// gspn_common.cuh — shared device-side definitions of the CUDA path (never used by oracle/).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gspn.h"

namespace gspn {

// Parameters of one gspn_fwd / gspn_bwd call as seen by every kernel (passed by value).
struct ScanParams {
  const void* x;    // [B,C,H,W]
  const void* wl;   // [D,B,G,H,W]
  const void* wm;
  const void* wr;
  const void* lam;  // [D,B,C,H,W]
  const void* h;    // bwd: saved forward output [D,B,C,H,W]
  const void* dh;   // bwd: upstream gradient   [D,B,C,H,W]
  void* hout;       // fwd output [D,B,C,H,W]
  void* dx;         // bwd outputs
  void* dwl;
  void* dwm;
  void* dwr;
  void* dlam;
  float* dx_acc;    // workspace: fp32 sum over directions [B,C,H,W]
  float* dwa_l;     // workspace: fp32 group sums of the normalised-tap gradients [D,B,G,H,W] (G < C)
  float* dwa_m;
  float* dwa_r;
  unsigned int* counters;  // workspace: completion counters (fast path)
  void* ws;                // bwd: caller workspace (carved by the launcher of the chosen path)
  size_t ws_bytes;
  int64_t B, C, H, W, G, D;
  int64_t kchunk;          // GSPN-local segment length along the scan axis (0: global scan)
  // merged backward (gspn_bwd_merged, NEXT-1): `dh` points at the gate u, the upstream gradient is
  // dh_d = merge_scale u_d dy, and du_d = merge_scale h_d dy is written to `du`
  const void* dy;          // [B,C,H,W]
  void* du;                // [D,B,C,H,W]
  float merge_scale;       // 1 (Sum) or 1/D (Mean)
  // recompute-h backward (NEXT-3): fp32 checkpoints of h every half-tile KS = 16 / s steps, per chain
  // [D,B,C][L/KS][P] (chain stride H W / KS): the forward writes them (and may skip h), the backward
  // recomputes each half-tile's h from them instead of reading h
  float* ckpt;
  uint32_t dirbit[4];      // direction bit (GSPN_DIR_*) of slab k
  uint32_t flags;
};

// Scan geometry of one direction inside an H x W plane: canonical offset of (t, r) is
// base + t * ts + r * rs (gspn.h direction table; R4).
struct DirGeom {
  int64_t L, P, base, ts, rs;
};

__host__ __device__ __forceinline__ DirGeom dir_geom(uint32_t dirbit, int64_t H, int64_t W) {
  DirGeom g;
  switch (dirbit) {
    case GSPN_DIR_T2B: g.L = H; g.P = W; g.base = 0;           g.ts = W;  g.rs = 1; break;
    case GSPN_DIR_B2T: g.L = H; g.P = W; g.base = (H - 1) * W; g.ts = -W; g.rs = 1; break;
    case GSPN_DIR_L2R: g.L = W; g.P = H; g.base = 0;           g.ts = 1;  g.rs = W; break;
    default:           g.L = W; g.P = H; g.base = W - 1;       g.ts = -1; g.rs = W; break;  // R2L
  }
  return g;
}

__device__ __forceinline__ bool is_vertical(uint32_t dirbit) {
  return dirbit == GSPN_DIR_T2B || dirbit == GSPN_DIR_B2T;
}

// GSPN-local (R19): segments of kchunk steps fixed on the canonical image grid
// (canonical scan-axis index s in segment s / kchunk, the last one short). A pixel starts its segment
// in scan order -- its h_{t-1} is not propagated -- when s % kchunk == 0 (T2B, L2R) or
// (s + 1) % kchunk == 0 or s is the last index (B2T, R2L). kchunk > 0.
__host__ __device__ __forceinline__ bool seg_start_px(uint32_t dirbit, int64_t i, int64_t j, int64_t H, int64_t W,
                                                      int64_t kchunk) {
  switch (dirbit) {
    case GSPN_DIR_T2B: return i % kchunk == 0;
    case GSPN_DIR_B2T: return (i + 1) % kchunk == 0 || i == H - 1;
    case GSPN_DIR_L2R: return j % kchunk == 0;
    default:           return (j + 1) % kchunk == 0 || j == W - 1;  // R2L
  }
}
// The same in scan coordinates: step t of a direction with scan length L (t = 0 always starts).
template <typename I>  // int64_t (generic path) or int (small planes: 32-bit modulo)
__host__ __device__ __forceinline__ bool seg_start_step(uint32_t dirbit, I t, I L, I kchunk) {
  if (t == 0) return true;
  if (kchunk <= 0) return false;
  const bool fwd_dir = dirbit == GSPN_DIR_T2B || dirbit == GSPN_DIR_L2R;
  return fwd_dir ? t % kchunk == 0 : (L - t) % kchunk == 0;  // reversed: canonical s = L-1-t
}

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Row-normalised taps of one position (R1/R2): out-of-range taps dropped,
// the in-range ones divided by their sum S. inv = 1/S (1 when the caller pre-normalised).
struct Taps {
  float a, b, c, inv;
};

__device__ __forceinline__ Taps make_taps(float wl, float wm, float wr, bool has_l, bool has_r, bool prenorm) {
  Taps t;
  const float l = has_l ? wl : 0.f;
  const float r = has_r ? wr : 0.f;
  if (prenorm) {
    t.a = l; t.b = wm; t.c = r; t.inv = 1.f;
  } else {
    t.inv = __frcp_rn(wm + l + r);
    t.a = l * t.inv; t.b = wm * t.inv; t.c = r * t.inv;
  }
  return t;
}

// Chain rule through the row normalisation (a, b, c) = (l, m, r) / S, S = l + m + r over the
// in-range raw taps (out-of-range taps are constant 0): with q = a Da + b Db + c Dc,
//   dw_l = (Da - q)/S = ((m + r) Da - m Db - r Dc) / S^2
//   dw_m = (Db - q)/S = ((l + r) Db - l Da - r Dc) / S^2
//   dw_r = (Dc - q)/S = ((l + m) Dc - l Da - m Db) / S^2
// The right-hand forms avoid the cancellation of q against D and are exactly 0 when only one tap is
// in range (P = 1). With pre-normalised taps the map is the identity on the in-range taps.
// kFastRcp: rcp.approx (<= 1 ulp) instead of the IEEE-rounded reciprocal (which carries a slow-path
// branch); the streaming kernels use it, the generic path keeps __frcp_rn.
template <bool kFastRcp = false>
__device__ __forceinline__ void jacobian(float wl, float wm, float wr, bool has_l, bool has_r, bool prenorm,
                                         float Da, float Db, float Dc, float& dwl, float& dwm, float& dwr) {
  const float l = has_l ? wl : 0.f;
  const float r = has_r ? wr : 0.f;
  if (prenorm) {
    dwl = has_l ? Da : 0.f; dwm = Db; dwr = has_r ? Dc : 0.f;
    return;
  }
  float inv;
  if constexpr (kFastRcp) asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(wm + l + r));
  else inv = __frcp_rn(wm + l + r);
  const float inv2 = inv * inv;
  dwl = has_l ? fmaf(wm + r, Da, -fmaf(wm, Db, r * Dc)) * inv2 : 0.f;
  dwm = fmaf(l + r, Db, -fmaf(l, Da, r * Dc)) * inv2;
  dwr = has_r ? fmaf(l + wm, Dc, -fmaf(l, Da, wm * Db)) * inv2 : 0.f;
}

}  // namespace gspn
