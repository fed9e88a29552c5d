/*
 * oracle/gspn_oracle.c — plain, slow, obviously-correct fp64 CPU oracle of the GSPN line scan.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this. The product path (paper_2512_07884_b200/) never links,
 * imports or calls it, and this file shares no code, header or table with the CUDA path.
 *
 * What it computes (the plain definition; every step in the paper's order and notation):
 *   PAPER.md:80-83 (§3.2, Eq. 1)      h_i = w_i h_{i-1} + Diag(lambda_i) x_i, per channel
 *   PAPER.md:144-146 (§4.2, Eq. 3)    the same recurrence with w_i shared by a group of channels
 *   PAPER.md:89 (§3.2)                w_i tridiagonal (3 neighbours of the previous row), row-stochastic,
 *                                     four directional passes T2B, B2T, L2R, R2L
 *   PAPER.md:155 (§4.2, Eq. 4)        first block row is Lambda_1, i.e. h_{-1} = 0
 *   PAPER.md:91-92 (§3.2)             GSPN-local: h resets at every kchunk segment start
 *   PAPER.md:84-88 (§3.2, Eq. 2)      output gate y = u (.) h, four passes combined (NEXT-1, merge_*)
 *   Backward: the adjoint (reverse-order) recurrence of the same linear map; the paper gives no
 *   formula, so this is the chain rule written out step by step.
 * Readings of silent points (R1-R16): row-stochastic = divide the in-range raw taps by
 * their sum; out-of-range taps dropped; w_l multiplies the smaller canonical parallel index; taps
 * stored at the output pixel; x shared by all directions; contiguous channel groups g = c / (C/G).
 *
 * Layout: x [B,C,H,W]; w_l,w_m,w_r [D,B,G,H,W]; lam,h,dh,dlam [D,B,C,H,W]; dx [B,C,H,W];
 * dw_* [D,B,G,H,W]; D = popcount(dirs), slabs in bit order T2B, B2T, L2R, R2L. All float64.
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared -pthread (no fast-math; no FMA contraction).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define T2B 1u
#define B2T 2u
#define L2R 4u
#define R2L 8u
#define PRENORMALIZED 1u

enum { ORACLE_OK = 0, ORACLE_BAD_ARG = 1, ORACLE_NONPOSITIVE_SUM = 5, ORACLE_NOMEM = 6 };

/* Detail of the last failed call. Workers write only their job's own buffer (under the job mutex);
 * run() copies it here after every worker has joined, so no two threads ever write g_detail. */
static char g_detail[256];

const char* gspn_oracle_detail(void) { return g_detail; }

/* Scan length L and parallel width P of a direction (gspn.h table). */
static void scan_shape(unsigned dir, int64_t H, int64_t W, int64_t* L, int64_t* P) {
  if (dir == T2B || dir == B2T) { *L = H; *P = W; } else { *L = W; *P = H; }
}

/* Canonical offset i*W + j of scan coordinate (t, r). */
static int64_t pixel(unsigned dir, int64_t H, int64_t W, int64_t t, int64_t r) {
  int64_t i = 0, j = 0;
  if (dir == T2B) { i = t; j = r; }
  else if (dir == B2T) { i = H - 1 - t; j = r; }
  else if (dir == L2R) { i = r; j = t; }
  else { i = r; j = W - 1 - t; }
  return i * W + j;
}

/* Normalised taps (a, b, c) at scan position r of width P from raw taps (wl, wm, wr).
 * Returns the row sum S through *S (1 when prenormalised). */
static int taps(double wl, double wm, double wr, int64_t r, int64_t P, unsigned flags,
                double* a, double* b, double* c, double* S) {
  const int has_l = (r >= 1), has_r = (r <= P - 2);
  if (flags & PRENORMALIZED) {
    *a = has_l ? wl : 0.0; *b = wm; *c = has_r ? wr : 0.0; *S = 1.0;
    return 0;
  }
  double s = wm;
  if (has_l) s += wl;
  if (has_r) s += wr;
  if (!(s > 0.0)) return 1;
  *a = has_l ? wl / s : 0.0;
  *b = wm / s;
  *c = has_r ? wr / s : 0.0;
  *S = s;
  return 0;
}

typedef struct {
  const double *x, *wl, *wm, *wr, *lam, *h, *dh;
  double *hout, *dx, *dwl, *dwm, *dwr, *dlam;
  int64_t B, C, H, W, G;
  int64_t kchunk; /* GSPN-local segment length along the scan axis; 0 = global scan */
  unsigned dirs, flags;
  int backward;
  int64_t next_unit; /* guarded by mu */
  pthread_mutex_t mu;
  int status;
  char detail[256]; /* first failure's detail, written under mu */
} job_t;

/* Records the first failing position of a job (thread-safe: under the job mutex). */
static void set_detail(job_t* J, unsigned dir, int64_t b, int64_t g, int64_t t, int64_t r) {
  pthread_mutex_lock(&J->mu);
  if (!J->detail[0])
    snprintf(J->detail, sizeof J->detail, "row sum S<=0 at dir=%u b=%lld g=%lld t=%lld r=%lld", dir, (long long)b,
             (long long)g, (long long)t, (long long)r);
  pthread_mutex_unlock(&J->mu);
}

static int dir_list(unsigned dirs, unsigned* out) {
  int n = 0;
  const unsigned all[4] = {T2B, B2T, L2R, R2L};
  for (int k = 0; k < 4; ++k) if (dirs & all[k]) out[n++] = all[k];
  return n;
}

/* GSPN-local (§3.2: "splits each row or column into fixed-length segments of size
 * kchunk and confines propagation to within those segments"; "At each kchunk segment
 * start, h resets to 0"). Segments are fixed on the canonical image grid -- canonical scan-axis index
 * s (row i for T2B/B2T, column j for L2R/R2L) lies in segment s / kchunk, the last one may be short
 * -- so all four directions confine propagation to the same image strips (DESIGN.md
 * R19). Returns 1 when scan step t of direction dir is the first step of its segment in scan order,
 * i.e. h_{t-1} does not reach h_t. kchunk = 0: the global scan, only t = 0 starts. */
static int seg_start(unsigned dir, int64_t t, int64_t L, int64_t kchunk) {
  if (t == 0) return 1;
  if (kchunk <= 0) return 0;
  if (dir == T2B || dir == L2R) return t % kchunk == 0;  /* canonical s = t */
  return (L - t) % kchunk == 0;                          /* canonical s = L-1-t: s + 1 multiple of kchunk */
}

/* Forward of unit (b, g): every channel of the group, every direction. Eq. 1 / Eq. 3 step by step. */
static int forward_unit(job_t* J, int64_t b, int64_t g) {
  const int64_t HW = J->H * J->W, Cg = J->C / J->G;
  unsigned dl[4];
  const int D = dir_list(J->dirs, dl);
  for (int k = 0; k < D; ++k) {
    int64_t L, P;
    scan_shape(dl[k], J->H, J->W, &L, &P);
    const double* wl = J->wl + ((int64_t)k * J->B * J->G + b * J->G + g) * HW;
    const double* wm = J->wm + ((int64_t)k * J->B * J->G + b * J->G + g) * HW;
    const double* wr = J->wr + ((int64_t)k * J->B * J->G + b * J->G + g) * HW;
    for (int64_t c = g * Cg; c < (g + 1) * Cg; ++c) {
      const double* x = J->x + (b * J->C + c) * HW;
      const double* lam = J->lam + ((int64_t)k * J->B * J->C + b * J->C + c) * HW;
      double* h = J->hout + ((int64_t)k * J->B * J->C + b * J->C + c) * HW;
      for (int64_t t = 0; t < L; ++t) {
        for (int64_t r = 0; r < P; ++r) {
          const int64_t p = pixel(dl[k], J->H, J->W, t, r);
          double a, bb, cc, S;
          if (taps(wl[p], wm[p], wr[p], r, P, J->flags, &a, &bb, &cc, &S)) {
            set_detail(J, dl[k], b, g, t, r);
            return ORACLE_NONPOSITIVE_SUM;
          }
          double acc = 0.0; /* w_i h_{i-1}: zero at t = 0 because h_{-1} = 0 */
          if (!seg_start(dl[k], t, L, J->kchunk)) { /* and at GSPN-local segment starts (h resets) */
            if (r >= 1) acc += a * h[pixel(dl[k], J->H, J->W, t - 1, r - 1)];
            acc += bb * h[pixel(dl[k], J->H, J->W, t - 1, r)];
            if (r <= P - 2) acc += cc * h[pixel(dl[k], J->H, J->W, t - 1, r + 1)];
          }
          h[p] = acc + lam[p] * x[p]; /* + Diag(lambda_i) x_i */
        }
      }
    }
  }
  return ORACLE_OK;
}

/* Backward of unit (b, g): the adjoint of forward_unit, reverse step order, given saved h. */
static int backward_unit(job_t* J, int64_t b, int64_t g) {
  const int64_t HW = J->H * J->W, Cg = J->C / J->G;
  unsigned dl[4];
  const int D = dir_list(J->dirs, dl);
  int64_t maxP = J->H > J->W ? J->H : J->W;
  double* gnext = (double*)calloc((size_t)maxP, sizeof(double));
  double* gcur = (double*)calloc((size_t)maxP, sizeof(double));
  double* Da = (double*)calloc((size_t)HW, sizeof(double));
  double* Db = (double*)calloc((size_t)HW, sizeof(double));
  double* Dc = (double*)calloc((size_t)HW, sizeof(double));
  int st = ORACLE_OK;
  if (!gnext || !gcur || !Da || !Db || !Dc) { st = ORACLE_NOMEM; goto done; }
  for (int64_t c = g * Cg; c < (g + 1) * Cg; ++c)
    memset(J->dx + (b * J->C + c) * HW, 0, (size_t)HW * sizeof(double));
  for (int k = 0; k < D; ++k) {
    int64_t L, P;
    scan_shape(dl[k], J->H, J->W, &L, &P);
    const int64_t wofs = ((int64_t)k * J->B * J->G + b * J->G + g) * HW;
    const double *wl = J->wl + wofs, *wm = J->wm + wofs, *wr = J->wr + wofs;
    memset(Da, 0, (size_t)HW * sizeof(double));
    memset(Db, 0, (size_t)HW * sizeof(double));
    memset(Dc, 0, (size_t)HW * sizeof(double));
    for (int64_t c = g * Cg; c < (g + 1) * Cg; ++c) {
      const int64_t cofs = ((int64_t)k * J->B * J->C + b * J->C + c) * HW;
      const double* x = J->x + (b * J->C + c) * HW;
      const double *lam = J->lam + cofs, *h = J->h + cofs, *dh = J->dh + cofs;
      double* dlam = J->dlam + cofs;
      double* dx = J->dx + (b * J->C + c) * HW;
      for (int64_t r = 0; r < P; ++r) gnext[r] = 0.0;
      for (int64_t t = L - 1; t >= 0; --t) {
        /* g_t = dh_t + w_{t+1}^T g_{t+1}  (adjoint of h_{t+1} = w_{t+1} h_t + ...) */
        for (int64_t r = 0; r < P; ++r) {
          double gt = dh[pixel(dl[k], J->H, J->W, t, r)];
          if (t + 1 < L && !seg_start(dl[k], t + 1, L, J->kchunk)) { /* h_{t+1} depends on h_t */
            double a, bb, cc, S;
            /* row r of w_{t+1} reaches h_t[r] through its centre tap */
            taps(wl[pixel(dl[k], J->H, J->W, t + 1, r)], wm[pixel(dl[k], J->H, J->W, t + 1, r)],
                 wr[pixel(dl[k], J->H, J->W, t + 1, r)], r, P, J->flags, &a, &bb, &cc, &S);
            gt += bb * gnext[r];
            if (r + 1 <= P - 1) { /* row r+1 reaches h_t[r] through its left tap */
              const int64_t q = pixel(dl[k], J->H, J->W, t + 1, r + 1);
              taps(wl[q], wm[q], wr[q], r + 1, P, J->flags, &a, &bb, &cc, &S);
              gt += a * gnext[r + 1];
            }
            if (r - 1 >= 0) { /* row r-1 reaches h_t[r] through its right tap */
              const int64_t q = pixel(dl[k], J->H, J->W, t + 1, r - 1);
              taps(wl[q], wm[q], wr[q], r - 1, P, J->flags, &a, &bb, &cc, &S);
              gt += cc * gnext[r - 1];
            }
          }
          gcur[r] = gt;
        }
        for (int64_t r = 0; r < P; ++r) {
          const int64_t p = pixel(dl[k], J->H, J->W, t, r);
          dlam[p] = gcur[r] * x[p]; /* d/dlambda of lambda_t x_t */
          dx[p] += gcur[r] * lam[p]; /* d/dx, summed over directions (R6) */
          if (!seg_start(dl[k], t, L, J->kchunk)) { /* d/d(normalised taps); zero where h_{t-1} is reset */
            if (r >= 1) Da[p] += gcur[r] * h[pixel(dl[k], J->H, J->W, t - 1, r - 1)];
            Db[p] += gcur[r] * h[pixel(dl[k], J->H, J->W, t - 1, r)];
            if (r <= P - 2) Dc[p] += gcur[r] * h[pixel(dl[k], J->H, J->W, t - 1, r + 1)];
          }
        }
        double* tmp = gnext; gnext = gcur; gcur = tmp;
      }
    }
    /* chain through the row normalisation a = w_l/S, b = w_m/S, c = w_r/S (sum over the group done) */
    double *dwl = J->dwl + wofs, *dwm = J->dwm + wofs, *dwr = J->dwr + wofs;
    for (int64_t t = 0; t < L; ++t) {
      for (int64_t r = 0; r < P; ++r) {
        const int64_t p = pixel(dl[k], J->H, J->W, t, r);
        double a, bb, cc, S;
        if (taps(wl[p], wm[p], wr[p], r, P, J->flags, &a, &bb, &cc, &S)) {
          set_detail(J, dl[k], b, g, t, r);
          st = ORACLE_NONPOSITIVE_SUM;
          goto done;
        }
        const int has_l = (r >= 1), has_r = (r <= P - 2);
        if (J->flags & PRENORMALIZED) {
          dwl[p] = has_l ? Da[p] : 0.0;
          dwm[p] = Db[p];
          dwr[p] = has_r ? Dc[p] : 0.0;
        } else {
          /* dL/dw_k = sum_j dL/dtap_j * dtap_j/dw_k = (Dtap_k - q) / S with q = a Da + b Db + c Dc */
          const double q = a * Da[p] + bb * Db[p] + cc * Dc[p];
          dwl[p] = has_l ? (Da[p] - q) / S : 0.0;
          dwm[p] = (Db[p] - q) / S;
          dwr[p] = has_r ? (Dc[p] - q) / S : 0.0;
        }
      }
    }
  }
done:
  free(gnext); free(gcur); free(Da); free(Db); free(Dc);
  return st;
}

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const int64_t u = J->next_unit++;
    const int bad = J->status;
    pthread_mutex_unlock(&J->mu);
    if (bad || u >= J->B * J->G) break;
    const int st = J->backward ? backward_unit(J, u / J->G, u % J->G) : forward_unit(J, u / J->G, u % J->G);
    if (st) {
      pthread_mutex_lock(&J->mu);
      if (!J->status) J->status = st;
      pthread_mutex_unlock(&J->mu);
    }
  }
  return NULL;
}

static int run(job_t* J, int threads) {
  if (J->B < 1 || J->C < 1 || J->H < 1 || J->W < 1 || J->G < 1 || J->C % J->G != 0 || J->dirs == 0 ||
      J->dirs > 15 || (J->flags & ~PRENORMALIZED) || J->kchunk < 0) {
    snprintf(g_detail, sizeof g_detail, "invalid argument");
    return ORACLE_BAD_ARG;
  }
  if (threads < 1) threads = 1;
  if (threads > 512) threads = 512;
  J->next_unit = 0;
  J->status = 0;
  pthread_mutex_init(&J->mu, NULL);
  pthread_t tid[512];
  int started = 0;
  for (int i = 1; i < threads; ++i)
    if (pthread_create(&tid[started], NULL, worker, J) == 0) ++started;
  worker(J);
  for (int i = 0; i < started; ++i) pthread_join(tid[i], NULL);
  pthread_mutex_destroy(&J->mu);
  if (J->status) memcpy(g_detail, J->detail, sizeof g_detail);
  return J->status;
}

int gspn_oracle_fwd(const double* x, const double* wl, const double* wm, const double* wr, const double* lam,
                    double* h, int64_t B, int64_t C, int64_t H, int64_t W, unsigned dirs, int64_t G,
                    unsigned flags, int64_t kchunk, int threads) {
  if (!x || !wl || !wm || !wr || !lam || !h) return ORACLE_BAD_ARG;
  job_t J;
  memset(&J, 0, sizeof J);
  J.x = x; J.wl = wl; J.wm = wm; J.wr = wr; J.lam = lam; J.hout = h;
  J.B = B; J.C = C; J.H = H; J.W = W; J.G = G; J.dirs = dirs; J.flags = flags; J.backward = 0;
  J.kchunk = kchunk;
  return run(&J, threads);
}

int gspn_oracle_bwd(const double* x, const double* wl, const double* wm, const double* wr, const double* lam,
                    const double* h, const double* dh, double* dx, double* dwl, double* dwm, double* dwr,
                    double* dlam, int64_t B, int64_t C, int64_t H, int64_t W, unsigned dirs, int64_t G,
                    unsigned flags, int64_t kchunk, int threads) {
  if (!x || !wl || !wm || !wr || !lam || !h || !dh || !dx || !dwl || !dwm || !dwr || !dlam) return ORACLE_BAD_ARG;
  job_t J;
  memset(&J, 0, sizeof J);
  J.x = x; J.wl = wl; J.wm = wm; J.wr = wr; J.lam = lam; J.h = h; J.dh = dh;
  J.dx = dx; J.dwl = dwl; J.dwm = dwm; J.dwr = dwr; J.dlam = dlam;
  J.B = B; J.C = C; J.H = H; J.W = W; J.G = G; J.dirs = dirs; J.flags = flags; J.backward = 1;
  J.kchunk = kchunk;
  return run(&J, threads);
}

/* Output gate and direction merge (§3.2 Eq. 2 "y = u (.) h", per direction; the four
 * directional passes are "combined" -- by Sum, or Mean on request, SPEC.md:203/263,
 * DESIGN.md R7):  y = s * sum_d u_d (.) h_d,  s = 1 (Sum) or 1/D (Mean).
 * h, u: [D, N] (N = B*C*H*W, direction slabs in bit order); y: [N]. */
void gspn_oracle_merge_fwd(const double* h, const double* u, double* y, int64_t D, int64_t N, int mean) {
  const double s = mean ? 1.0 / (double)D : 1.0;
  for (int64_t n = 0; n < N; ++n) {
    double acc = 0.0;
    for (int64_t d = 0; d < D; ++d) acc += u[d * N + n] * h[d * N + n];
    y[n] = s * acc;
  }
}

/* Its adjoint: dh_d = s * u_d (.) dy,  du_d = s * h_d (.) dy  (y is bilinear in (u, h)). */
void gspn_oracle_merge_bwd(const double* h, const double* u, const double* dy, double* dh, double* du, int64_t D,
                           int64_t N, int mean) {
  const double s = mean ? 1.0 / (double)D : 1.0;
  for (int64_t d = 0; d < D; ++d)
    for (int64_t n = 0; n < N; ++n) {
      dh[d * N + n] = s * (u[d * N + n] * dy[n]);
      du[d * N + n] = s * (h[d * N + n] * dy[n]);
    }
}

/* Compact-channel proxy projections (§4.2 "project the input tensor x in R^{N x C x H x W}
 * into a lower-dimensional proxy subspace x_proxy in R^{N x C_proxy x H x W}"; "expand back
 * to C with a learned 1x1 projection"). A 1x1 convolution is a channel mix at every
 * pixel:  out[b, o, n] = sum_i M[o, i] in[b, i, n]   (n over the H W pixels; M [Co, Ci] row-major).
 * Down-projection: M = P_down [C_proxy, C]; up-projection: M = P_up [C, C_proxy]. Its adjoints are the
 * same mix with M^T (d in) and the weight gradient dM[o, i] = sum_{b, n} d out[b, o, n] in[b, i, n]. */
void gspn_oracle_proxy_mix(const double* in, const double* M, double* out, int64_t B, int64_t Ci, int64_t Co,
                           int64_t HW) {
  for (int64_t b = 0; b < B; ++b)
    for (int64_t o = 0; o < Co; ++o)
      for (int64_t n = 0; n < HW; ++n) {
        double acc = 0.0;
        for (int64_t i = 0; i < Ci; ++i) acc += M[o * Ci + i] * in[(b * Ci + i) * HW + n];
        out[(b * Co + o) * HW + n] = acc;
      }
}

void gspn_oracle_proxy_wgrad(const double* dout, const double* in, double* dM, int64_t B, int64_t Ci, int64_t Co,
                             int64_t HW) {
  for (int64_t o = 0; o < Co; ++o)
    for (int64_t i = 0; i < Ci; ++i) {
      double acc = 0.0;
      for (int64_t b = 0; b < B; ++b)
        for (int64_t n = 0; n < HW; ++n) acc += dout[(b * Co + o) * HW + n] * in[(b * Ci + i) * HW + n];
      dM[o * Ci + i] = acc;
    }
}
