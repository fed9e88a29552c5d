// gspn_api.cu — the C ABI declared in include/gspn.h: host-side validation (before any CUDA call),
// workspace carving, path selection (TMA streaming fast path, else the generic path) and launch.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <exception>

#include "gspn_internal.h"

namespace {

thread_local char t_detail[512] = "";
thread_local const char* t_path = "none";
thread_local int t_launches = 0;

gspn_status_t fail(gspn_status_t st, const char* fmt, const char* what, long long v = 0) {
  snprintf(t_detail, sizeof t_detail, fmt, what, v);
  return st;
}

int popcount4(uint32_t d) { return (d & 1) + ((d >> 1) & 1) + ((d >> 2) & 1) + ((d >> 3) & 1); }

struct Span {
  const char* name;
  uintptr_t lo, hi;
};

bool overlap(const Span& a, const Span& b) { return a.lo < b.hi && b.lo < a.hi; }

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// Common dimension checks. Returns GSPN_OK or GSPN_ERR_INVALID_ARG with the detail set.
gspn_status_t check_dims(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t G, gspn_dtype_t dt,
                         uint32_t flags) {
  if (B < 1) return fail(GSPN_ERR_INVALID_ARG, "%s must be >= 1 (got %lld)", "B", B);
  if (C < 1) return fail(GSPN_ERR_INVALID_ARG, "%s must be >= 1 (got %lld)", "C", C);
  if (H < 1) return fail(GSPN_ERR_INVALID_ARG, "%s must be >= 1 (got %lld)", "H", H);
  if (W < 1) return fail(GSPN_ERR_INVALID_ARG, "%s must be >= 1 (got %lld)", "W", W);
  if (G < 1) return fail(GSPN_ERR_INVALID_ARG, "%s must be >= 1 (got %lld)", "groups", G);
  if (C % G != 0) return fail(GSPN_ERR_INVALID_ARG, "%s: C %% groups != 0 (groups=%lld)", "groups", G);
  if (dirs == 0 || dirs > 15) return fail(GSPN_ERR_INVALID_ARG, "%s must be in [1, 15] (got %lld)", "dirs", dirs);
  if (dt != GSPN_F32 && dt != GSPN_BF16) return fail(GSPN_ERR_INVALID_ARG, "%s unknown (%lld)", "dtype", (long long)dt);
  if (flags & ~(GSPN_FLAG_PRENORMALIZED | GSPN_FLAG_FORCE_GENERIC | GSPN_FLAG_FORCE_SPLIT | GSPN_FLAG_DW_F32))
    return fail(GSPN_ERR_INVALID_ARG, "%s has unknown bits (0x%llx)", "flags", flags);
  // Overflow guard: the largest tensor (D*B*C*H*W elements) must stay far below 2^62 bytes, and the
  // chain count must fit a 1-D grid.
  const double n = (double)popcount4(dirs) * (double)B * (double)C * (double)H * (double)W * 4.0;
  if (n >= 4.0e18) return fail(GSPN_ERR_INVALID_ARG, "%s: tensor too large (%lld elements per plane)", "shape", H * W);
  if ((double)popcount4(dirs) * (double)B * (double)C >= 2147483647.0)
    return fail(GSPN_ERR_INVALID_ARG, "%s: D*B*C chains exceed 2^31-1 (B*C=%lld)", "shape", B * C);
  return GSPN_OK;
}

gspn_status_t check_ptr(const void* p, const char* name) {
  if (p == nullptr) {
    snprintf(t_detail, sizeof t_detail, "%s is NULL", name);
    return GSPN_ERR_INVALID_ARG;
  }
  if (reinterpret_cast<uintptr_t>(p) % 16 != 0) {
    snprintf(t_detail, sizeof t_detail, "%s is not 16-byte aligned", name);
    return GSPN_ERR_INVALID_ARG;
  }
  return GSPN_OK;
}

gspn_status_t check_aliasing(const Span* outs, int n_out, const Span* ins, int n_in) {
  for (int i = 0; i < n_out; ++i) {
    for (int j = 0; j < n_in; ++j)
      if (overlap(outs[i], ins[j])) {
        snprintf(t_detail, sizeof t_detail, "output %s overlaps input %s", outs[i].name, ins[j].name);
        return GSPN_ERR_INVALID_ARG;
      }
    for (int j = i + 1; j < n_out; ++j)
      if (overlap(outs[i], outs[j])) {
        snprintf(t_detail, sizeof t_detail, "output %s overlaps output %s", outs[i].name, outs[j].name);
        return GSPN_ERR_INVALID_ARG;
      }
  }
  return GSPN_OK;
}

Span span(const char* name, const void* p, size_t bytes) {
  return Span{name, reinterpret_cast<uintptr_t>(p), reinterpret_cast<uintptr_t>(p) + bytes};
}

void fill_dirs(gspn::ScanParams& p, uint32_t dirs) {
  int k = 0;
  const uint32_t order[4] = {GSPN_DIR_T2B, GSPN_DIR_B2T, GSPN_DIR_L2R, GSPN_DIR_R2L};
  for (int i = 0; i < 4; ++i)
    if (dirs & order[i]) p.dirbit[k++] = order[i];
  for (; k < 4; ++k) p.dirbit[k] = 0;
}

size_t generic_workspace(int64_t B, int64_t C, int64_t H, int64_t W, int64_t D, int64_t G) {
  size_t n = align_up((size_t)(B * C * H * W) * sizeof(float));                  // dx_acc
  if (G < C) n += 3 * align_up((size_t)(D * B * G * H * W) * sizeof(float));     // dwa_l/m/r
  return n;
}

}  // namespace

extern "C" {

const char* gspn_status_string(gspn_status_t s) {
  switch (s) {
    case GSPN_OK: return "GSPN_OK";
    case GSPN_ERR_INVALID_ARG: return "GSPN_ERR_INVALID_ARG";
    case GSPN_ERR_UNSUPPORTED: return "GSPN_ERR_UNSUPPORTED";
    case GSPN_ERR_CUDA: return "GSPN_ERR_CUDA";
    case GSPN_ERR_INTERNAL: return "GSPN_ERR_INTERNAL";
  }
  return "GSPN_ERR_UNKNOWN";
}

const char* gspn_last_error_detail(void) { return t_detail; }
const char* gspn_last_path(void) { return t_path; }
int gspn_last_launch_count(void) { return t_launches; }

double gspn_algorithmic_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                              gspn_dtype_t dtype, int backward) {
  if (check_dims(B, C, H, W, dirs, groups, dtype, 0) != GSPN_OK) return 0.0;
  const double s = dtype == GSPN_BF16 ? 2.0 : 4.0;
  const double D = popcount4(dirs);
  const double N = (double)B * C * H * W, Nw = (double)B * groups * H * W;
  const double fwd = s * (N * (1.0 + 2.0 * D) + 3.0 * D * Nw);
  return backward ? 2.0 * fwd : fwd;
}

size_t gspn_bwd_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                                gspn_dtype_t dtype) {
  if (check_dims(B, C, H, W, dirs, groups, dtype, 0) != GSPN_OK) return 0;
  const int64_t D = popcount4(dirs);
  size_t a = generic_workspace(B, C, H, W, D, groups);
  size_t b = gspn::stream_bwd_workspace_bytes(B, C, H, W, D, groups, dtype);
  return a > b ? a : b;
}

gspn_status_t gspn_fwd(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam, void* h,
                       int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                       gspn_dtype_t dtype, uint32_t flags, gspn_stream_t stream) {
  return gspn_fwd_local(x, w_l, w_m, w_r, lam, h, B, C, H, W, dirs, groups, 0, dtype, flags, stream);
}

gspn_status_t gspn_fwd_local(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                             void* h, int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                             int64_t kchunk, gspn_dtype_t dtype, uint32_t flags, gspn_stream_t stream) {
  try {
    gspn_status_t st;
    if (kchunk < 0) return fail(GSPN_ERR_INVALID_ARG, "%s must be >= 0 (got %lld)", "kchunk", kchunk);
    if ((st = check_ptr(x, "x")) || (st = check_ptr(w_l, "w_l")) || (st = check_ptr(w_m, "w_m")) ||
        (st = check_ptr(w_r, "w_r")) || (st = check_ptr(lam, "lam")) || (st = check_ptr(h, "h")))
      return st;
    if ((st = check_dims(B, C, H, W, dirs, groups, dtype, flags))) return st;
    const int64_t D = popcount4(dirs);
    const size_t s = dtype == GSPN_BF16 ? 2 : 4;
    const size_t nx = (size_t)(B * C * H * W) * s, nl = (size_t)D * nx, nw = (size_t)(D * B * groups * H * W) * s;
    const Span ins[5] = {span("x", x, nx), span("w_l", w_l, nw), span("w_m", w_m, nw), span("w_r", w_r, nw),
                         span("lam", lam, nl)};
    const Span outs[1] = {span("h", h, nl)};
    if ((st = check_aliasing(outs, 1, ins, 5))) return st;
    if (H > gspn::generic_max_P() || W > gspn::generic_max_P()) {
      snprintf(t_detail, sizeof t_detail, "H or W above %lld is not tiled", (long long)gspn::generic_max_P());
      return GSPN_ERR_UNSUPPORTED;
    }

    gspn::ScanParams p;
    memset(&p, 0, sizeof p);
    p.x = x; p.wl = w_l; p.wm = w_m; p.wr = w_r; p.lam = lam; p.hout = h;
    p.B = B; p.C = C; p.H = H; p.W = W; p.G = groups; p.D = D; p.flags = flags;
    p.kchunk = kchunk >= (H > W ? H : W) ? 0 : kchunk;  // a segment covering every scan is the global scan
    fill_dirs(p, dirs);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    int launches = 0;
    bool handled = false;
    cudaError_t e = cudaSuccess;
    const char* path = "generic";
    if (!(flags & GSPN_FLAG_FORCE_GENERIC)) {
      const char* spath = "stream";
      e = gspn::launch_fwd_stream(p, dtype, cs, &launches, &handled, &spath);
      if (handled) path = spath;
      if (e == cudaSuccess && !handled && gspn::small_eligible(p)) {
        e = gspn::launch_fwd_small(p, dtype, cs, &launches);
        handled = true;
        path = "small";
      }
    }
    if (e == cudaSuccess && !handled) e = gspn::launch_fwd_generic(p, dtype, cs, &launches);
    if (e != cudaSuccess) {
      snprintf(t_detail, sizeof t_detail, "CUDA error: %s", cudaGetErrorString(e));
      return GSPN_ERR_CUDA;
    }
    t_path = path;
    t_launches = launches;
    return GSPN_OK;
  } catch (const std::exception& ex) {
    snprintf(t_detail, sizeof t_detail, "internal: %s", ex.what());
    return GSPN_ERR_INTERNAL;
  } catch (...) {
    snprintf(t_detail, sizeof t_detail, "internal error");
    return GSPN_ERR_INTERNAL;
  }
}

gspn_status_t gspn_bwd(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                       const void* h, const void* dh, void* dx, void* dw_l, void* dw_m, void* dw_r, void* dlam,
                       int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                       gspn_dtype_t dtype, uint32_t flags, void* workspace, size_t workspace_bytes,
                       gspn_stream_t stream) {
  return gspn_bwd_local(x, w_l, w_m, w_r, lam, h, dh, dx, dw_l, dw_m, dw_r, dlam, B, C, H, W, dirs, groups, 0, dtype,
                        flags, workspace, workspace_bytes, stream);
}

gspn_status_t gspn_bwd_local(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                             const void* h, const void* dh, void* dx, void* dw_l, void* dw_m, void* dw_r, void* dlam,
                             int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                             int64_t kchunk, gspn_dtype_t dtype, uint32_t flags, void* workspace,
                             size_t workspace_bytes, gspn_stream_t stream) {
  try {
    gspn_status_t st;
    if (kchunk < 0) return fail(GSPN_ERR_INVALID_ARG, "%s must be >= 0 (got %lld)", "kchunk", kchunk);
    if ((st = check_ptr(x, "x")) || (st = check_ptr(w_l, "w_l")) || (st = check_ptr(w_m, "w_m")) ||
        (st = check_ptr(w_r, "w_r")) || (st = check_ptr(lam, "lam")) || (st = check_ptr(h, "h")) ||
        (st = check_ptr(dh, "dh")) || (st = check_ptr(dx, "dx")) || (st = check_ptr(dw_l, "dw_l")) ||
        (st = check_ptr(dw_m, "dw_m")) || (st = check_ptr(dw_r, "dw_r")) || (st = check_ptr(dlam, "dlam")))
      return st;
    if ((st = check_dims(B, C, H, W, dirs, groups, dtype, flags))) return st;
    const int64_t D = popcount4(dirs);
    const size_t need = gspn_bwd_workspace_bytes(B, C, H, W, dirs, groups, dtype);
    if (need > 0) {
      if ((st = check_ptr(workspace, "workspace"))) return st;
      if (workspace_bytes < need) {
        snprintf(t_detail, sizeof t_detail, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
        return GSPN_ERR_INVALID_ARG;
      }
    }
    if ((flags & GSPN_FLAG_DW_F32) && groups == C) {
      snprintf(t_detail, sizeof t_detail, "GSPN_FLAG_DW_F32 needs groups < C (got groups == C == %lld)", (long long)C);
      return GSPN_ERR_UNSUPPORTED;
    }
    const size_t s = dtype == GSPN_BF16 ? 2 : 4;
    const size_t sw = (flags & GSPN_FLAG_DW_F32) ? 4 : s;  // dw element size
    const size_t nx = (size_t)(B * C * H * W) * s, nl = (size_t)D * nx, nw = (size_t)(D * B * groups * H * W) * s;
    const size_t nwo = (size_t)(D * B * groups * H * W) * sw;
    const Span ins[7] = {span("x", x, nx),   span("w_l", w_l, nw), span("w_m", w_m, nw), span("w_r", w_r, nw),
                         span("lam", lam, nl), span("h", h, nl),     span("dh", dh, nl)};
    Span outs[6] = {span("dx", dx, nx),     span("dw_l", dw_l, nwo), span("dw_m", dw_m, nwo),
                    span("dw_r", dw_r, nwo), span("dlam", dlam, nl), span("workspace", workspace, need)};
    if ((st = check_aliasing(outs, need > 0 ? 6 : 5, ins, 7))) return st;
    if (H > gspn::generic_max_P() || W > gspn::generic_max_P()) {
      snprintf(t_detail, sizeof t_detail, "H or W above %lld is not tiled", (long long)gspn::generic_max_P());
      return GSPN_ERR_UNSUPPORTED;
    }

    gspn::ScanParams p;
    memset(&p, 0, sizeof p);
    p.x = x; p.wl = w_l; p.wm = w_m; p.wr = w_r; p.lam = lam; p.h = h; p.dh = dh;
    p.dx = dx; p.dwl = dw_l; p.dwm = dw_m; p.dwr = dw_r; p.dlam = dlam;
    p.B = B; p.C = C; p.H = H; p.W = W; p.G = groups; p.D = D; p.flags = flags;
    p.kchunk = kchunk >= (H > W ? H : W) ? 0 : kchunk;
    fill_dirs(p, dirs);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    int launches = 0;
    bool handled = false;
    cudaError_t e = cudaSuccess;
    const char* stream_path = "stream";
    if (!(flags & GSPN_FLAG_FORCE_GENERIC)) {
      // the streaming path carves the workspace itself
      p.ws = workspace;
      p.ws_bytes = workspace_bytes;
      e = gspn::launch_bwd_stream(p, dtype, cs, &launches, &handled, &stream_path);
    }
    if (e == cudaSuccess && !handled) {
      char* ws = static_cast<char*>(workspace);
      p.dx_acc = reinterpret_cast<float*>(ws);
      const size_t dx_bytes = align_up((size_t)(B * C * H * W) * sizeof(float));
      size_t off = dx_bytes;
      const size_t zero_bytes = generic_workspace(B, C, H, W, D, groups);
      if (groups < C) {
        const size_t nwb = align_up((size_t)(D * B * groups * H * W) * sizeof(float));
        p.dwa_l = reinterpret_cast<float*>(ws + off); off += nwb;
        p.dwa_m = reinterpret_cast<float*>(ws + off); off += nwb;
        p.dwa_r = reinterpret_cast<float*>(ws + off); off += nwb;
      }
      if (!(flags & GSPN_FLAG_FORCE_GENERIC) && gspn::small_eligible(p) && gspn::small_grouped(p, dtype)) {
        // small planes, grouped weights: taps once per group, dw formed in-kernel, one launch
        stream_path = "small";
        handled = true;
        e = gspn::launch_bwd_small_grouped(p, dtype, cs, &launches);
      } else if (!(flags & GSPN_FLAG_FORCE_GENERIC) && gspn::small_eligible(p)) {
        // small-plane path: dx summed inside the CTA; only the group sums (G < C) use the workspace
        stream_path = "small";
        handled = true;
        if (groups < C) e = cudaMemsetAsync(ws + dx_bytes, 0, zero_bytes - dx_bytes, cs);
        if (e == cudaSuccess) e = gspn::launch_bwd_small(p, dtype, cs, &launches);
        if (e == cudaSuccess && groups < C) e = gspn::launch_finish_dw(p, dtype, cs, &launches);
      } else {
        e = cudaMemsetAsync(workspace, 0, zero_bytes, cs);
        if (e == cudaSuccess) e = gspn::launch_bwd_generic(p, dtype, cs, &launches);
      }
    }
    if (e != cudaSuccess) {
      snprintf(t_detail, sizeof t_detail, "CUDA error: %s", cudaGetErrorString(e));
      return GSPN_ERR_CUDA;
    }
    t_path = handled ? stream_path : "generic";
    t_launches = launches;
    return GSPN_OK;
  } catch (const std::exception& ex) {
    snprintf(t_detail, sizeof t_detail, "internal: %s", ex.what());
    return GSPN_ERR_INTERNAL;
  } catch (...) {
    snprintf(t_detail, sizeof t_detail, "internal error");
    return GSPN_ERR_INTERNAL;
  }
}

}  // extern "C"

namespace {

// Shared validation of the merge entry points (dims, dirs, dtype, flags).
gspn_status_t check_merge(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, gspn_dtype_t dt, uint32_t flags) {
  if (flags & ~GSPN_FLAG_MERGE_MEAN) return fail(GSPN_ERR_INVALID_ARG, "%s has unknown bits (0x%llx)", "flags", flags);
  return check_dims(B, C, H, W, dirs, 1, dt, 0);
}

template <typename F>
gspn_status_t guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& ex) {
    snprintf(t_detail, sizeof t_detail, "internal: %s", ex.what());
    return GSPN_ERR_INTERNAL;
  } catch (...) {
    snprintf(t_detail, sizeof t_detail, "internal error");
    return GSPN_ERR_INTERNAL;
  }
}

}  // namespace

// The proxy kernels index pixels and (batch, channel) pairs in 32-bit: reject extents beyond INT32_MAX
// instead of letting the casts truncate (offsets themselves are formed in 64-bit).
static gspn_status_t check_proxy_extent(int64_t B, int64_t Ci, int64_t Co, int64_t H, int64_t W) {
  const int64_t lim = INT32_MAX;
  if (H > lim / W) return fail(GSPN_ERR_UNSUPPORTED, "%s: H*W above INT32_MAX (H = %lld)", "shape", H);
  if (B > lim / std::max(Ci, Co) || Ci > lim / Co)
    return fail(GSPN_ERR_UNSUPPORTED, "%s: B*C or Ci*Co above INT32_MAX", "shape");
  return GSPN_OK;
}

extern "C" {

size_t gspn_ckpt_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                       gspn_dtype_t dtype) {
  if (check_dims(B, C, H, W, dirs, groups, dtype, 0) != GSPN_OK) return 0;
  const int64_t KS = dtype == GSPN_BF16 ? 8 : 4;  // one fp32 checkpoint per half-tile of KS steps
  const int64_t L = (H > W ? H : W);
  return align_up((size_t)popcount4(dirs) * (size_t)(B * C) * (size_t)(((L + KS - 1) / KS) * L) * sizeof(float));
}

size_t gspn_bwd_recompute_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                                          gspn_dtype_t dtype) {
  const size_t a = gspn_bwd_workspace_bytes(B, C, H, W, dirs, groups, dtype);
  if (check_dims(B, C, H, W, dirs, groups, dtype, 0) != GSPN_OK) return 0;
  const size_t s = dtype == GSPN_BF16 ? 2 : 4;
  return align_up(a) + align_up((size_t)popcount4(dirs) * (size_t)(B * C * H * W) * s);  // + h (fallback)
}

static void scan_params(gspn::ScanParams& p, const void* x, const void* w_l, const void* w_m, const void* w_r,
                        const void* lam, int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                        uint32_t flags) {
  memset(&p, 0, sizeof p);
  p.x = x; p.wl = w_l; p.wm = w_m; p.wr = w_r; p.lam = lam;
  p.B = B; p.C = C; p.H = H; p.W = W; p.G = groups; p.D = popcount4(dirs); p.flags = flags;
  fill_dirs(p, dirs);
}

gspn_status_t gspn_fwd_ckpt(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                            void* h, float* ckpt, int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs,
                            int64_t groups, gspn_dtype_t dtype, uint32_t flags, gspn_stream_t stream) {
  return guarded([&]() -> gspn_status_t {
    gspn_status_t st;
    if ((st = check_ptr(x, "x")) || (st = check_ptr(w_l, "w_l")) || (st = check_ptr(w_m, "w_m")) ||
        (st = check_ptr(w_r, "w_r")) || (st = check_ptr(lam, "lam")) || (st = check_ptr(ckpt, "ckpt")))
      return st;
    if (h != nullptr && (st = check_ptr(h, "h"))) return st;
    if (flags & ~(GSPN_FLAG_PRENORMALIZED | GSPN_FLAG_FORCE_GENERIC))
      return fail(GSPN_ERR_INVALID_ARG, "%s has unknown bits (0x%llx)", "flags", flags);
    if ((st = check_dims(B, C, H, W, dirs, groups, dtype, flags))) return st;
    const size_t s = dtype == GSPN_BF16 ? 2 : 4;
    const int64_t D = popcount4(dirs);
    const size_t nx = (size_t)(B * C * H * W) * s, nl = (size_t)D * nx, nw = (size_t)(D * B * groups * H * W) * s;
    const Span ins[5] = {span("x", x, nx), span("w_l", w_l, nw), span("w_m", w_m, nw), span("w_r", w_r, nw),
                         span("lam", lam, nl)};
    const Span outs[2] = {span("ckpt", ckpt, gspn_ckpt_bytes(B, C, H, W, dirs, groups, dtype)),
                          span("h", h ? h : ckpt, h ? nl : 0)};
    if ((st = check_aliasing(outs, h ? 2 : 1, ins, 5))) return st;
    if (H > gspn::generic_max_P() || W > gspn::generic_max_P())
      return fail(GSPN_ERR_UNSUPPORTED, "%s above the tiled maximum (%lld)", "H or W", (long long)gspn::generic_max_P());
    gspn::ScanParams p;
    scan_params(p, x, w_l, w_m, w_r, lam, B, C, H, W, dirs, groups, flags);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    int launches = 0;
    cudaError_t e = cudaSuccess;
    const char* path;
    if (!(flags & GSPN_FLAG_FORCE_GENERIC) && gspn::ckpt_eligible(p, dtype)) {
      p.hout = h;
      p.ckpt = ckpt;
      bool handled = false;
      const char* spath = nullptr;
      e = gspn::launch_fwd_stream(p, dtype, cs, &launches, &handled, &spath);
      if (e == cudaSuccess && !handled) e = cudaErrorNotSupported;
      path = "stream-ckpt";
    } else if (h != nullptr) {  // no checkpoints on this path: the recompute backward re-runs the forward
      const gspn_status_t sf = gspn_fwd(x, w_l, w_m, w_r, lam, h, B, C, H, W, dirs, groups, dtype, flags, stream);
      if (sf != GSPN_OK) return sf;
      launches = t_launches;
      path = "ckpt-deferred";
    } else {
      path = "ckpt-deferred";  // nothing to keep: the backward recomputes h from the inputs
    }
    if (e != cudaSuccess) {
      snprintf(t_detail, sizeof t_detail, "CUDA error: %s", cudaGetErrorString(e));
      return GSPN_ERR_CUDA;
    }
    t_path = path;
    t_launches = launches;
    return GSPN_OK;
  });
}

gspn_status_t gspn_bwd_recompute(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                                 const float* ckpt, const void* dh, void* dx, void* dw_l, void* dw_m, void* dw_r,
                                 void* dlam, int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs,
                                 int64_t groups, gspn_dtype_t dtype, uint32_t flags, void* workspace,
                                 size_t workspace_bytes, gspn_stream_t stream) {
  return guarded([&]() -> gspn_status_t {
    gspn_status_t st;
    if ((st = check_ptr(x, "x")) || (st = check_ptr(w_l, "w_l")) || (st = check_ptr(w_m, "w_m")) ||
        (st = check_ptr(w_r, "w_r")) || (st = check_ptr(lam, "lam")) || (st = check_ptr(ckpt, "ckpt")) ||
        (st = check_ptr(dh, "dh")) || (st = check_ptr(dx, "dx")) || (st = check_ptr(dw_l, "dw_l")) ||
        (st = check_ptr(dw_m, "dw_m")) || (st = check_ptr(dw_r, "dw_r")) || (st = check_ptr(dlam, "dlam")))
      return st;
    if (flags & ~(GSPN_FLAG_PRENORMALIZED | GSPN_FLAG_FORCE_GENERIC))
      return fail(GSPN_ERR_INVALID_ARG, "%s has unknown bits (0x%llx)", "flags", flags);
    if ((st = check_dims(B, C, H, W, dirs, groups, dtype, flags))) return st;
    const size_t need_bwd = gspn_bwd_workspace_bytes(B, C, H, W, dirs, groups, dtype);
    const size_t need = gspn_bwd_recompute_workspace_bytes(B, C, H, W, dirs, groups, dtype);
    if ((st = check_ptr(workspace, "workspace"))) return st;
    if (workspace_bytes < need) {
      snprintf(t_detail, sizeof t_detail, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
      return GSPN_ERR_INVALID_ARG;
    }
    const size_t s = dtype == GSPN_BF16 ? 2 : 4;
    const int64_t D = popcount4(dirs);
    const size_t nx = (size_t)(B * C * H * W) * s, nl = (size_t)D * nx, nw = (size_t)(D * B * groups * H * W) * s;
    const Span ins[7] = {span("x", x, nx),     span("w_l", w_l, nw), span("w_m", w_m, nw), span("w_r", w_r, nw),
                         span("lam", lam, nl), span("dh", dh, nl),
                         span("ckpt", ckpt, gspn_ckpt_bytes(B, C, H, W, dirs, groups, dtype))};
    const Span outs[6] = {span("dx", dx, nx),     span("dw_l", dw_l, nw), span("dw_m", dw_m, nw),
                          span("dw_r", dw_r, nw), span("dlam", dlam, nl), span("workspace", workspace, need)};
    if ((st = check_aliasing(outs, 6, ins, 7))) return st;
    gspn::ScanParams p;
    scan_params(p, x, w_l, w_m, w_r, lam, B, C, H, W, dirs, groups, flags);
    p.dh = dh; p.dx = dx; p.dwl = dw_l; p.dwm = dw_m; p.dwr = dw_r; p.dlam = dlam;
    p.ckpt = const_cast<float*>(ckpt);
    p.ws = workspace;
    p.ws_bytes = need_bwd;
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    int launches = 0;
    cudaError_t e = cudaSuccess;
    const char* path = "stream-recompute";
    bool handled = false;
    if (!(flags & GSPN_FLAG_FORCE_GENERIC) && H <= gspn::generic_max_P() && W <= gspn::generic_max_P())
      handled = gspn::launch_bwd_recompute(p, dtype, cs, &launches, &e);
    if (!handled) {  // no checkpoints for this shape: the whole forward again (h into the workspace), then gspn_bwd
      path = "recompute-unfused";
      void* hws = static_cast<char*>(workspace) + align_up(need_bwd);
      gspn_status_t sf = gspn_fwd(x, w_l, w_m, w_r, lam, hws, B, C, H, W, dirs, groups, dtype, flags, stream);
      if (sf != GSPN_OK) return sf;
      launches = t_launches;
      sf = gspn_bwd(x, w_l, w_m, w_r, lam, hws, dh, dx, dw_l, dw_m, dw_r, dlam, B, C, H, W, dirs, groups, dtype, flags,
                    workspace, need_bwd, stream);
      if (sf != GSPN_OK) return sf;
      launches += t_launches;
    }
    if (e != cudaSuccess) {
      snprintf(t_detail, sizeof t_detail, "CUDA error: %s", cudaGetErrorString(e));
      return GSPN_ERR_CUDA;
    }
    t_path = path;
    t_launches = launches;
    return GSPN_OK;
  });
}

size_t gspn_fwd_merged_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                                       gspn_dtype_t dtype) {
  if (check_dims(B, C, H, W, dirs, groups, dtype, 0) != GSPN_OK) return 0;
  const size_t s = dtype == GSPN_BF16 ? 2 : 4;
  return align_up((size_t)popcount4(dirs) * (size_t)(B * C * H * W) * s);  // h, when the caller keeps none
}

gspn_status_t gspn_fwd_merged(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                              const void* u, void* h, void* y, int64_t B, int64_t C, int64_t H, int64_t W,
                              uint32_t dirs, int64_t groups, gspn_dtype_t dtype, uint32_t flags, void* workspace,
                              size_t workspace_bytes, gspn_stream_t stream) {
  return guarded([&]() -> gspn_status_t {
    gspn_status_t st;
    if ((st = check_ptr(x, "x")) || (st = check_ptr(w_l, "w_l")) || (st = check_ptr(w_m, "w_m")) ||
        (st = check_ptr(w_r, "w_r")) || (st = check_ptr(lam, "lam")) || (st = check_ptr(u, "u")) ||
        (st = check_ptr(y, "y")))
      return st;
    if (flags & ~(GSPN_FLAG_PRENORMALIZED | GSPN_FLAG_MERGE_MEAN | GSPN_FLAG_FORCE_GENERIC))
      return fail(GSPN_ERR_INVALID_ARG, "%s has unknown bits (0x%llx)", "flags", flags);
    const uint32_t sflags = flags & ~GSPN_FLAG_MERGE_MEAN;
    if ((st = check_dims(B, C, H, W, dirs, groups, dtype, sflags))) return st;
    const int64_t D = popcount4(dirs);
    const size_t s = dtype == GSPN_BF16 ? 2 : 4;
    const size_t nx = (size_t)(B * C * H * W) * s, nl = (size_t)D * nx, nw = (size_t)(D * B * groups * H * W) * s;
    void* hh = h;
    if (hh == nullptr) {  // h lives in the workspace
      if ((st = check_ptr(workspace, "workspace"))) return st;
      if (workspace_bytes < nl) {
        snprintf(t_detail, sizeof t_detail, "workspace too small: %zu < %zu bytes", workspace_bytes, nl);
        return GSPN_ERR_INVALID_ARG;
      }
      hh = workspace;
    } else if ((st = check_ptr(h, "h"))) {
      return st;
    }
    const Span ins[6] = {span("x", x, nx),     span("w_l", w_l, nw), span("w_m", w_m, nw),
                         span("w_r", w_r, nw), span("lam", lam, nl), span("u", u, nl)};
    const Span outs[2] = {span(h ? "h" : "workspace", hh, nl), span("y", y, nx)};
    if ((st = check_aliasing(outs, 2, ins, 6))) return st;
    if (H > gspn::generic_max_P() || W > gspn::generic_max_P())
      return fail(GSPN_ERR_UNSUPPORTED, "%s above the tiled maximum (%lld)", "H or W", (long long)gspn::generic_max_P());
    const bool mean = (flags & GSPN_FLAG_MERGE_MEAN) != 0;
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    int launches = 0;
    bool handled = false;
    cudaError_t e = cudaSuccess;
    const char* path = "stream-merged";
    if (!(flags & GSPN_FLAG_FORCE_GENERIC)) {
      gspn::ScanParams p;
      memset(&p, 0, sizeof p);
      p.x = x; p.wl = w_l; p.wm = w_m; p.wr = w_r; p.lam = lam; p.hout = hh;
      p.B = B; p.C = C; p.H = H; p.W = W; p.G = groups; p.D = D; p.flags = sflags;
      fill_dirs(p, dirs);
      e = gspn::launch_fwd_merged(p, dtype, u, y, mean ? 1.f / static_cast<float>(D) : 1.f, cs, &launches, &handled);
    }
    if (e == cudaSuccess && !handled) {  // the scan, then the merge
      path = "merged-unfused";
      const gspn_status_t sf = gspn_fwd(x, w_l, w_m, w_r, lam, hh, B, C, H, W, dirs, groups, dtype, sflags, stream);
      if (sf != GSPN_OK) return sf;
      launches = t_launches + 1;
      e = gspn::launch_merge_fwd(hh, u, y, B * C * H * W, static_cast<int>(D), mean, dtype, cs);
    }
    if (e != cudaSuccess) {
      snprintf(t_detail, sizeof t_detail, "CUDA error: %s", cudaGetErrorString(e));
      return GSPN_ERR_CUDA;
    }
    t_path = path;
    t_launches = launches;
    return GSPN_OK;
  });
}

size_t gspn_bwd_merged_workspace_bytes(int64_t B, int64_t C, int64_t H, int64_t W, uint32_t dirs, int64_t groups,
                                       gspn_dtype_t dtype) {
  const size_t a = gspn_bwd_workspace_bytes(B, C, H, W, dirs, groups, dtype);
  if (a == 0 && check_dims(B, C, H, W, dirs, groups, dtype, 0) != GSPN_OK) return 0;
  const size_t s = dtype == GSPN_BF16 ? 2 : 4;
  return align_up(a) + align_up((size_t)popcount4(dirs) * (size_t)(B * C * H * W) * s);  // + dh (unfused fallback)
}

gspn_status_t gspn_bwd_merged(const void* x, const void* w_l, const void* w_m, const void* w_r, const void* lam,
                              const void* h, const void* u, const void* dy, void* dx, void* dw_l, void* dw_m,
                              void* dw_r, void* dlam, void* du, int64_t B, int64_t C, int64_t H, int64_t W,
                              uint32_t dirs, int64_t groups, gspn_dtype_t dtype, uint32_t flags, void* workspace,
                              size_t workspace_bytes, gspn_stream_t stream) {
  return guarded([&]() -> gspn_status_t {
    gspn_status_t st;
    if ((st = check_ptr(x, "x")) || (st = check_ptr(w_l, "w_l")) || (st = check_ptr(w_m, "w_m")) ||
        (st = check_ptr(w_r, "w_r")) || (st = check_ptr(lam, "lam")) || (st = check_ptr(h, "h")) ||
        (st = check_ptr(u, "u")) || (st = check_ptr(dy, "dy")) || (st = check_ptr(dx, "dx")) ||
        (st = check_ptr(dw_l, "dw_l")) || (st = check_ptr(dw_m, "dw_m")) || (st = check_ptr(dw_r, "dw_r")) ||
        (st = check_ptr(dlam, "dlam")) || (st = check_ptr(du, "du")))
      return st;
    if (flags & ~(GSPN_FLAG_PRENORMALIZED | GSPN_FLAG_MERGE_MEAN | GSPN_FLAG_FORCE_GENERIC))
      return fail(GSPN_ERR_INVALID_ARG, "%s has unknown bits (0x%llx)", "flags", flags);
    const uint32_t sflags = flags & ~GSPN_FLAG_MERGE_MEAN;
    if ((st = check_dims(B, C, H, W, dirs, groups, dtype, sflags))) return st;
    const int64_t D = popcount4(dirs);
    const size_t need_bwd = gspn_bwd_workspace_bytes(B, C, H, W, dirs, groups, dtype);
    const size_t need = gspn_bwd_merged_workspace_bytes(B, C, H, W, dirs, groups, dtype);
    if ((st = check_ptr(workspace, "workspace"))) return st;
    if (workspace_bytes < need) {
      snprintf(t_detail, sizeof t_detail, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
      return GSPN_ERR_INVALID_ARG;
    }
    const size_t s = dtype == GSPN_BF16 ? 2 : 4;
    const size_t nx = (size_t)(B * C * H * W) * s, nl = (size_t)D * nx, nw = (size_t)(D * B * groups * H * W) * s;
    const Span ins[8] = {span("x", x, nx),     span("w_l", w_l, nw), span("w_m", w_m, nw), span("w_r", w_r, nw),
                         span("lam", lam, nl), span("h", h, nl),     span("u", u, nl),     span("dy", dy, nx)};
    const Span outs[7] = {span("dx", dx, nx),     span("dw_l", dw_l, nw), span("dw_m", dw_m, nw),
                          span("dw_r", dw_r, nw), span("dlam", dlam, nl), span("du", du, nl),
                          span("workspace", workspace, need)};
    if ((st = check_aliasing(outs, 7, ins, 8))) return st;
    const bool mean = (flags & GSPN_FLAG_MERGE_MEAN) != 0;
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    int launches = 0;
    bool handled = false;
    cudaError_t e = cudaSuccess;
    const char* path = "stream-fused-merged";
    if (!(flags & GSPN_FLAG_FORCE_GENERIC) && H <= gspn::generic_max_P() && W <= gspn::generic_max_P()) {
      gspn::ScanParams p;
      memset(&p, 0, sizeof p);
      p.x = x; p.wl = w_l; p.wm = w_m; p.wr = w_r; p.lam = lam; p.h = h; p.dh = u;
      p.dx = dx; p.dwl = dw_l; p.dwm = dw_m; p.dwr = dw_r; p.dlam = dlam;
      p.dy = dy; p.du = du; p.merge_scale = mean ? 1.f / static_cast<float>(D) : 1.f;
      p.B = B; p.C = C; p.H = H; p.W = W; p.G = groups; p.D = D; p.flags = sflags;
      fill_dirs(p, dirs);
      p.ws = workspace;
      p.ws_bytes = need_bwd;
      const char* spath = nullptr;
      e = gspn::launch_bwd_stream(p, dtype, cs, &launches, &handled, &spath);
    }
    if (e == cudaSuccess && !handled) {
      // unfused: dh = s u dy (and du) by the merge adjoint into the workspace, then the plain backward
      path = "merged-unfused";
      void* dh = static_cast<char*>(workspace) + align_up(need_bwd);
      e = gspn::launch_merge_bwd(h, u, dy, dh, du, B * C * H * W, static_cast<int>(D), mean, dtype, cs);
      if (e == cudaSuccess) {
        const gspn_status_t sb = gspn_bwd(x, w_l, w_m, w_r, lam, h, dh, dx, dw_l, dw_m, dw_r, dlam, B, C, H, W, dirs,
                                          groups, dtype, sflags, workspace, need_bwd, stream);
        if (sb != GSPN_OK) return sb;
        launches = 1 + t_launches;
      }
    }
    if (e != cudaSuccess) {
      snprintf(t_detail, sizeof t_detail, "CUDA error: %s", cudaGetErrorString(e));
      return GSPN_ERR_CUDA;
    }
    t_path = path;
    t_launches = launches;
    return GSPN_OK;
  });
}

gspn_status_t gspn_merge_fwd(const void* h, const void* u, void* y, int64_t B, int64_t C, int64_t H, int64_t W,
                             uint32_t dirs, gspn_dtype_t dtype, uint32_t flags, gspn_stream_t stream) {
  return guarded([&]() -> gspn_status_t {
    gspn_status_t st;
    if ((st = check_ptr(h, "h")) || (st = check_ptr(u, "u")) || (st = check_ptr(y, "y"))) return st;
    if ((st = check_merge(B, C, H, W, dirs, dtype, flags))) return st;
    const int D = popcount4(dirs);
    const size_t s = dtype == GSPN_BF16 ? 2 : 4;
    const int64_t N = B * C * H * W;
    const Span ins[2] = {span("h", h, (size_t)D * N * s), span("u", u, (size_t)D * N * s)};
    const Span outs[1] = {span("y", y, (size_t)N * s)};
    if ((st = check_aliasing(outs, 1, ins, 2))) return st;
    const cudaError_t e = gspn::launch_merge_fwd(h, u, y, N, D, flags & GSPN_FLAG_MERGE_MEAN, dtype,
                                                 reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) {
      snprintf(t_detail, sizeof t_detail, "CUDA error: %s", cudaGetErrorString(e));
      return GSPN_ERR_CUDA;
    }
    t_path = "merge";
    t_launches = 1;
    return GSPN_OK;
  });
}

gspn_status_t gspn_merge_bwd(const void* h, const void* u, const void* dy, void* dh, void* du, int64_t B, int64_t C,
                             int64_t H, int64_t W, uint32_t dirs, gspn_dtype_t dtype, uint32_t flags,
                             gspn_stream_t stream) {
  return guarded([&]() -> gspn_status_t {
    gspn_status_t st;
    if ((st = check_ptr(h, "h")) || (st = check_ptr(u, "u")) || (st = check_ptr(dy, "dy")) ||
        (st = check_ptr(dh, "dh")) || (st = check_ptr(du, "du")))
      return st;
    if ((st = check_merge(B, C, H, W, dirs, dtype, flags))) return st;
    const int D = popcount4(dirs);
    const size_t s = dtype == GSPN_BF16 ? 2 : 4;
    const int64_t N = B * C * H * W;
    const Span ins[3] = {span("h", h, (size_t)D * N * s), span("u", u, (size_t)D * N * s),
                         span("dy", dy, (size_t)N * s)};
    const Span outs[2] = {span("dh", dh, (size_t)D * N * s), span("du", du, (size_t)D * N * s)};
    if ((st = check_aliasing(outs, 2, ins, 3))) return st;
    const cudaError_t e = gspn::launch_merge_bwd(h, u, dy, dh, du, N, D, flags & GSPN_FLAG_MERGE_MEAN, dtype,
                                                 reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) {
      snprintf(t_detail, sizeof t_detail, "CUDA error: %s", cudaGetErrorString(e));
      return GSPN_ERR_CUDA;
    }
    t_path = "merge";
    t_launches = 1;
    return GSPN_OK;
  });
}


gspn_status_t gspn_proxy_mix(const void* in, const void* M, void* out, int64_t B, int64_t Ci, int64_t Co, int64_t H,
                             int64_t W, gspn_dtype_t dtype, uint32_t flags, gspn_stream_t stream) {
  return guarded([&]() -> gspn_status_t {
    gspn_status_t st;
    if ((st = check_ptr(in, "in")) || (st = check_ptr(M, "M")) || (st = check_ptr(out, "out"))) return st;
    if (flags & ~(GSPN_FLAG_PROXY_TRANSPOSE | GSPN_FLAG_PROXY_SIMT))
      return fail(GSPN_ERR_INVALID_ARG, "%s has unknown bits (0x%llx)", "flags", flags);
    if ((st = check_dims(B, Ci, H, W, 1, 1, dtype, 0))) return st;
    if (Co < 1) return fail(GSPN_ERR_INVALID_ARG, "%s must be >= 1 (got %lld)", "Co", Co);
    if ((H * W) % 2 != 0) return fail(GSPN_ERR_UNSUPPORTED, "%s: H*W must be even (got %lld)", "shape", H * W);
    if ((st = check_proxy_extent(B, Ci, Co, H, W))) return st;
    // tcgen05 (TMEM accumulator, TMA-streamed activations) for bf16 shapes it tiles; SIMT otherwise
    const bool umma = !(flags & GSPN_FLAG_PROXY_SIMT) && gspn::umma_mix_eligible(B, Ci, Co, H * W, dtype);
    if (!umma && Ci * Co > 49152) return fail(GSPN_ERR_UNSUPPORTED, "%s: Co*Ci above 49152 (%lld)", "M", Ci * Co);
    const size_t s = dtype == GSPN_BF16 ? 2 : 4;
    const Span ins[2] = {span("in", in, (size_t)(B * Ci * H * W) * s), span("M", M, (size_t)(Ci * Co) * s)};
    const Span outs[1] = {span("out", out, (size_t)(B * Co * H * W) * s)};
    if ((st = check_aliasing(outs, 1, ins, 2))) return st;
    const cudaError_t e =
        umma ? gspn::launch_umma_mix(in, M, out, B, Ci, Co, H * W, flags & GSPN_FLAG_PROXY_TRANSPOSE,
                                     reinterpret_cast<cudaStream_t>(stream))
             : gspn::launch_proxy_mix(in, M, out, B, Ci, Co, H * W, flags & GSPN_FLAG_PROXY_TRANSPOSE, dtype,
                                      reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) {
      snprintf(t_detail, sizeof t_detail, "CUDA error: %s", cudaGetErrorString(e));
      return GSPN_ERR_CUDA;
    }
    t_path = umma ? "proxy-umma" : "proxy";
    t_launches = 1;
    return GSPN_OK;
  });
}

gspn_status_t gspn_proxy_wgrad(const void* dout, const void* in, float* dM, int64_t B, int64_t Ci, int64_t Co,
                               int64_t H, int64_t W, gspn_dtype_t dtype, gspn_stream_t stream) {
  return guarded([&]() -> gspn_status_t {
    gspn_status_t st;
    if ((st = check_ptr(dout, "dout")) || (st = check_ptr(in, "in")) || (st = check_ptr(dM, "dM"))) return st;
    if ((st = check_dims(B, Ci, H, W, 1, 1, dtype, 0))) return st;
    if (Co < 1) return fail(GSPN_ERR_INVALID_ARG, "%s must be >= 1 (got %lld)", "Co", Co);
    if ((st = check_proxy_extent(B, Ci, Co, H, W))) return st;
    const bool umma = gspn::umma_wgrad_eligible(B, Ci, Co, H * W, dtype);
    if (!umma && (Co + Ci) * 33 + Co * Ci > 49152)
      return fail(GSPN_ERR_UNSUPPORTED, "%s: (Co+Ci)*33 + Co*Ci above 49152 (Co*Ci = %lld)", "shape", Ci * Co);
    const size_t s = dtype == GSPN_BF16 ? 2 : 4;
    const Span ins[2] = {span("dout", dout, (size_t)(B * Co * H * W) * s), span("in", in, (size_t)(B * Ci * H * W) * s)};
    const Span outs[1] = {span("dM", dM, (size_t)(Ci * Co) * sizeof(float))};
    if ((st = check_aliasing(outs, 1, ins, 2))) return st;
    const cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (umma) {  // tcgen05: per-CTA partial sums in TMEM, added into the zeroed fp32 dM
      e = cudaMemsetAsync(dM, 0, (size_t)(Ci * Co) * sizeof(float), cs);
      if (e == cudaSuccess) e = gspn::launch_umma_wgrad(dout, in, dM, B, Ci, Co, H * W, cs);
    } else {
      e = gspn::launch_proxy_wgrad(dout, in, dM, B, Ci, Co, H * W, dtype, cs);
    }
    if (e != cudaSuccess) {
      snprintf(t_detail, sizeof t_detail, "CUDA error: %s", cudaGetErrorString(e));
      return GSPN_ERR_CUDA;
    }
    t_path = umma ? "proxy-umma" : "proxy";
    t_launches = 1;
    return GSPN_OK;
  });
}

}  // extern "C"
