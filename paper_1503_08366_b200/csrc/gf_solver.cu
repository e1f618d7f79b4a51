// ADMM graph-projection-splitting iteration (reference solver.py:248-437).
//
// Data layout in HBM (per rank, tall problems m >= n, row partition):
//   A_hat    m x ld   working dtype T (fp32/fp64), scaled in place by setup
//   Ginv     q x ldq  T, (I + A_hat' A_hat)^-1, q = n
//   x side   n-vectors fp64: x^, x~, c_x, x_1/2 [2], mu^_1/2 [2]  (+ T copies of
//            x^, x^_1/2 and rhs as the GEMV right-hand sides)
//   y side   m-vectors fp64: y^, y~, c_y, y_1/2 [2], nu^_1/2 [2]
// The half iterates are double-buffered by iteration parity so a degenerate
// iteration can hand back the previous one (solver.py:337-342).
//
// A tall iteration k is three launches (programmatic dependent launch between
// them when no communicator is active):
//   S(k-1) x+ = G^-1 rhs on a TMA row ring (gf_ring.cuh) with the whole x side
//          in the epilogue: x~ update, prox_g of iteration k, mu^_1/2, c_x,
//          ||mu||, g(x) partials.
//   F(k)   the fused single pass over A_hat (gf_fused.cuh): row pass
//          A_hat [x^, x^_1/2] with the whole y side in the epilogue -- y~
//          update (dual step + adaptive-rho rescale of k-1), prox_f, nu^_1/2,
//          c_y, r_pri / ||y|| / f(y) partials (r_pri = ||D^-1 (A_hat x^_1/2 -
//          y^_1/2)||) -- and, while each row is still in shared memory, the
//          column pass A_hat' [c_y, nu^_1/2] into per-CTA slabs.
//   Z(k)   slab and record reductions (+ NCCL all-reduce of [2n + 8] under a
//          row partition), rhs = c_x + A_hat' c_y, r_dual =
//          ||E^-1 (A_hat' nu^ + mu^)||, and in the last CTA the controller:
//          stop rule (solver.py:191-202, 373-376), degenerate checks, history
//          row, adaptive rho (solver.py:221-239).
// Rows too wide for the fused ring (and wide problems) use the two-pass
// schedule: a row pass with the y side, then a column pass,
// which reads A_hat twice; the unscaled A is never touched.
// The controller lives on the device, so a chunk of iterations runs without a
// host round trip; kernels of iterations after termination return at entry.

#include <mutex>
#include <vector>

#include "gf_internal.h"
#include "gf_gemv.cuh"
#include "gf_fused.cuh"
#include "gf_ring.cuh"
#include "gf_sym.cuh"

#include <cudaTypedefs.h>

namespace gf {

struct Ctl {
  int status;
  unsigned ticket;
  unsigned zflags;     // non-finite flags raised by the controller kernel's CTAs
  unsigned pad_;
  int64_t k;           // iteration being assembled (R/C/Z) / prepared (S)
  int64_t iterations;  // SolveResult.iterations once terminated
  int64_t last_good;   // last recorded iteration, -1 if none
  int64_t l_mark, u_mark;
  int64_t inner;       // CGLS inner iterations of the last projection
  double rho, rho_prev, ratio, final_rho;
  double r_pri, r_dual, eps_pri, eps_dual, objective;
  double gap;          // duality gap of the last gap test (solver.py:378-390)
  int64_t gap_set;     // 1 once a gap was computed
  unsigned gcnt, ggen; // grid barrier of the fused pass's Z tail (arrivals, generation)
  unsigned scnt, sgen; // grid barrier of the lower-triangle G^-1 GEMV (gf_sym.cuh)
};

struct Params {
  double abs_tol, rel_tol, alpha, delta, tau;
  int64_t max_iter;
  int adaptive;
  int gap;             // gap-based stopping on (and every conjugate supported)
};

// per-row / per-column reductions (+ a flags word):
//   y: r_pri^2, ||y||^2, f(y), drift_y^2, f(y_full), f*(nu_full)
//   x: ||mu||^2, g(x), drift_x^2, g(x_full), g*(mu_full)
// the last two of each are the duality gap at the full iterate (gap_stop only)
constexpr int kRedY = 6;
constexpr int kRedX = 5;
constexpr int kScal = 8;  // all-reduced scalars after the 2*ld column sums
enum : unsigned { kBadXPlus = 1, kBadXHalf = 2, kBadYPlus = 4, kBadYHalf = 8 };

template <typename T>
struct YEpi {
  static constexpr int NR = kRedY;
  Ctl* ctl;
  TermsView f;
  const double* d;
  double *yk, *yt, *cy, *yh2, *nuh2;
  int64_t m;
  double alpha;
  int warm_x;
  int gap;
  // controller scalars, cached in registers by begin() (fused kernel)
  int64_t k_ = -1;
  double rho_ = 0.0, ratio_ = 1.0;
  __device__ bool active() const { return ctl->status == GF_STATUS_RUNNING; }
  __device__ void begin() {
    k_ = ctl->k;
    rho_ = ctl->rho;
    ratio_ = ctl->ratio;
  }
  __device__ void row(int64_t i, const double* dots, double* red, unsigned& flags) const {
    double w0, w1;
    row_w(i, dots, red, flags, w0, w1);
  }
  // Per-row inputs of the epilogue, loadable ahead of the dot products.
  struct RowIn {
    double di, cy, yk, yt;
    Term t;
  };
  __device__ RowIn load_in(int64_t i) const {
    RowIn in;
    in.di = d[i];
    in.cy = cy[i];
    in.yk = yk[i];
    in.yt = yt[i];
    in.t = load_term(f, i);
    return in;
  }
  // w0 = c_y_i, w1 = nu^_1/2_i: the column-pass weights of this row.
  __device__ void row_w(int64_t i, const double* dots, double* red, unsigned& flags, double& w0,
                        double& w1) const {
    finish(i, load_in(i), dots, red, flags, w0, w1);
  }
  // The fused kernel splits the epilogue at the column-pass weights: mid()
  // is the critical path (the compute warps wait for w0, w1), tail() the
  // stores and reductions that run after the hand-off.
  struct Mid {
    int64_t k;
    double rho, ykv, ytv, yh, yhh, nu, cyn;
  };
  __device__ Mid mid(const RowIn& in, const double* dots, double& w0, double& w1) const {
    const bool cached = k_ >= 0;
    Mid r;
    r.k = cached ? k_ : ctl->k;
    const double rho = cached ? rho_ : ctl->rho;
    r.rho = rho;
    if (r.k == 0) {
      r.ykv = warm_x ? dots[0] : in.yk;
      r.ytv = in.yt;
    } else {
      r.ykv = dots[0];                        // y+ = A_hat x+  (projection.py:122)
      r.ytv = M_(S_(in.cy, r.ykv), cached ? ratio_ : ctl->ratio);   // y~ + r_y - y+, rescaled (solver.py:420, :237)
    }
    const double di = in.di;
    r.yh = prox_term(in.t, M_(rho, M_(di, di)), D_(S_(r.ykv, r.ytv), di));  // solver.py:331-336
    r.yhh = M_(r.yh, di);
    r.nu = M_(-rho, A_(S_(r.yhh, r.ykv), r.ytv));                            // solver.py:180
    const double ry = A_(M_(alpha, r.yhh), M_(S_(1.0, alpha), r.ykv));      // solver.py:394
    r.cyn = A_(ry, r.ytv);
    w0 = r.cyn;
    w1 = r.nu;
    return r;
  }
  __device__ void tail(int64_t i, const RowIn& in, const double* dots, const Mid& r, double* red,
                       unsigned& flags) const {
    if (!isfinite(r.ykv)) flags |= kBadYPlus;
    if (!isfinite(r.yh)) flags |= kBadYHalf;
    const int64_t b = (r.k & 1) * m;
    yk[i] = r.ykv;
    yt[i] = r.ytv;
    yh2[b + i] = r.yh;
    nuh2[b + i] = r.nu;
    cy[i] = r.cyn;
    const double rp = S_(D_(dots[1], in.di), r.yh);   // (A x_1/2 - y_1/2)_i via A_hat
    red[0] += rp * rp;
    red[1] += r.yh * r.yh;
    red[2] += eval_term(in.t, r.yh);
    red[3] += (r.yhh - r.ykv) * (r.yhh - r.ykv);
    if (gap) {   // full iterate y = y^ / d, nu = -rho d y~ (solver.py:379-382)
      bool unsup = false;
      red[4] += eval_term(in.t, D_(r.ykv, in.di));
      red[5] += conj_term(in.t, M_(M_(-r.rho, in.di), r.ytv), unsup);
    }
  }
  __device__ void finish(int64_t i, const RowIn& in, const double* dots, double* red, unsigned& flags,
                         double& w0, double& w1) const {
    tail(i, in, dots, mid(in, dots, w0, w1), red, flags);
  }
};

template <typename T>
struct XEpi {
  static constexpr int NR = kRedX;
  Ctl* ctl;
  TermsView g;
  const double* e;
  double *xk, *xt, *cx, *xh2, *muh2;
  T *xk_T, *xh_T;   // row-pass right-hand sides: [x^ (tall) or c_x (wide), x^_1/2]
  int64_t n;
  double alpha;
  int wide;          // wide orientation: the first right-hand side is c_x
  int gap;
  __device__ bool active() const { return ctl->status == GF_STATUS_RUNNING; }
  // init: x^, x~ given (warm start or zero) -- iteration 0 has no dual step.
  __device__ void apply(int64_t j, double xkv, double xtv, double* red, unsigned& flags) const {
    const int64_t k1 = ctl->k;
    const double rho = ctl->rho;
    const double ej = e[j];
    const Term t = load_term(g, j);
    const double xh = prox_term(t, D_(rho, M_(ej, ej)), M_(ej, S_(xkv, xtv)));   // solver.py:330-335
    if (!isfinite(xh)) flags |= kBadXHalf;
    const double xhh = D_(xh, ej);
    const double mu = M_(-rho, A_(S_(xhh, xkv), xtv));                   // solver.py:179
    const double rx = A_(M_(alpha, xhh), M_(S_(1.0, alpha), xkv));      // solver.py:393
    const int64_t b = (k1 & 1) * n;
    xk[j] = xkv;
    xt[j] = xtv;
    xh2[b + j] = xh;
    muh2[b + j] = mu;
    cx[j] = A_(rx, xtv);
    xk_T[j] = (T)(wide ? A_(rx, xtv) : xkv);
    xh_T[j] = (T)xhh;
    const double mo = D_(mu, ej);
    red[0] += mo * mo;
    red[1] += eval_term(t, xh);
    red[2] += (xhh - xkv) * (xhh - xkv);
    if (gap) {   // full iterate x = e x^, mu = -rho x~ / e (solver.py:379-382)
      bool unsup = false;
      red[3] += eval_term(t, M_(ej, xkv));
      red[4] += conj_term(t, D_(M_(-rho, xtv), ej), unsup);
    }
  }
  __device__ void row(int64_t j, const double* dots, double* red, unsigned& flags) const {
    const double xp = dots[0];                                           // x+ (projection.py:121)
    if (!isfinite(xp)) flags |= kBadXPlus;
    apply(j, xp, M_(S_(cx[j], xp), ctl->ratio), red, flags);            // solver.py:419, :237
  }
};

// ---------------------------------------------------------- wide (m < n) --
// Row pass of the wide schedule: dots = [A_hat c_x, A_hat x^_1/2]; the y side
// of iteration k (its y^ is the y+ of the previous projection, kept in ypl)
// and the projection right-hand side A c - d (projection.py:124).
template <typename T>
struct YEpiW {
  static constexpr int NR = kRedY;
  Ctl* ctl;
  TermsView f;
  const double* d;
  double *yk, *yt, *cy, *yh2, *nuh2;
  const double* ypl;
  T* rhs_T;
  int64_t m;
  double alpha;
  int gap;
  __device__ bool active() const { return ctl->status == GF_STATUS_RUNNING; }
  __device__ void row(int64_t i, const double* dots, double* red, unsigned& flags) const {
    const int64_t k = ctl->k;
    const double rho = ctl->rho;
    double ykv, ytv;
    if (k == 0) {
      ykv = yk[i];
      ytv = yt[i];
    } else {
      ykv = ypl[i];                                           // y+ of projection k-1
      ytv = M_(S_(cy[i], ykv), ctl->ratio);                   // solver.py:420, :237
    }
    const double di = d[i];
    const Term t = load_term(f, i);
    const double yh = prox_term(t, M_(rho, M_(di, di)), D_(S_(ykv, ytv), di));
    if (!isfinite(yh)) flags |= kBadYHalf;
    const double yhh = M_(yh, di);
    const double nu = M_(-rho, A_(S_(yhh, ykv), ytv));
    const double ry = A_(M_(alpha, yhh), M_(S_(1.0, alpha), ykv));
    const double cyn = A_(ry, ytv);
    const int64_t b = (k & 1) * m;
    yk[i] = ykv;
    yt[i] = ytv;
    yh2[b + i] = yh;
    nuh2[b + i] = nu;
    cy[i] = cyn;
    rhs_T[i] = (T)S_(dots[0], cyn);                           // A c - d
    const double rp = S_(D_(dots[1], di), yh);
    red[0] += rp * rp;
    red[1] += yh * yh;
    red[2] += eval_term(t, yh);
    red[3] += (yhh - ykv) * (yhh - ykv);
    if (gap) {
      bool unsup = false;
      red[4] += eval_term(t, D_(ykv, di));
      red[5] += conj_term(t, M_(M_(-rho, di), ytv), unsup);
    }
  }
};

// Ginv pass of the wide schedule: w = (I + A A')^-1 (A c - d), y+ = d + w.
struct WEpi {
  static constexpr int NR = 0;
  Ctl* ctl;
  const double* cy;
  double *w, *ypl;
  __device__ bool active() const { return ctl->status == GF_STATUS_RUNNING; }
  __device__ void row(int64_t i, const double* dots, double*, unsigned& flags) const {
    w[i] = dots[0];
    const double yp = A_(cy[i], dots[0]);                     // projection.py:125
    ypl[i] = yp;
    if (!isfinite(yp)) flags |= kBadYPlus;
  }
};

// Indirect wide step: the CGLS tolerance schedule needs the drift of
// iteration k, sqrt(||x^_1/2 - x^||^2 + ||y^_1/2 - y^||^2) (solver.py:401-405),
// before the controller runs: from the R(k) records and the x records of
// X(k-1) / x-init.  out = [drift, status].
__global__ void wide_drift_kernel(const Ctl* __restrict__ ctl, const double* __restrict__ rpart, int64_t nr,
                                  const double* __restrict__ xpart, int64_t nx, double* __restrict__ out) {
  __shared__ double sh[8];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) s += rpart[i * (kRedY + 1) + 3];
  for (int64_t i = threadIdx.x; i < nx; i += blockDim.x) s += xpart[i * (kRedX + 1) + 2];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    out[0] = sqrt(t);
    out[1] = (double)ctl->status;
  }
}

// After the wide CGLS (w = z in place): y+ = c_y + w (projection.py:161) and
// its finiteness flags, one word per CTA in the WEpi record layout.
__global__ void __launch_bounds__(256) wide_cgls_finish_kernel(const double* __restrict__ cy,
                                                               const double* __restrict__ w, double* __restrict__ ypl,
                                                               int64_t m, double* __restrict__ spart) {
  unsigned flags = 0;
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const double yp = A_(cy[i], w[i]);
    ypl[i] = yp;
    if (!isfinite(yp)) flags |= kBadYPlus;
  }
  flags = warp_or(flags);
  __shared__ unsigned sf[8];
  if ((threadIdx.x & 31) == 0) sf[threadIdx.x >> 5] = flags;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned f = 0;
    for (int i = 0; i < 8; ++i) f |= sf[i];
    spart[blockIdx.x] = (double)f;
  }
}

__global__ void neg_diff_kernel(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                                double* __restrict__ neg_b, int64_t n) {
  // out = a - b, neg_b = -b
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = S_(a[i], b[i]);
    neg_b[i] = -b[i];
  }
}

// x side after the controller from an x+ given as a vector: wide schedule
// x+ = c_x - A_hat' w (projection.py:126, sub = 1), or the CGLS solution of
// the indirect mode (projection.py:148-150, sub = 0); then the dual step and
// prox_g of iteration k+1.
// xk_prev / xt_prev (wide only, may be null) keep x^ and x~ of the iteration
// just recorded, which this kernel overwrites with those of the next one: a
// trace snapshot of iteration k reads them (solver.py:362-367).
template <typename T>
__global__ void __launch_bounds__(256) x_wide_kernel(XEpi<T> epi, const double* __restrict__ aw,
                                                     double* __restrict__ part, int sub, double* __restrict__ xk_prev,
                                                     double* __restrict__ xt_prev) {
  if (!epi.active()) return;
  double red[kRedX] = {};
  unsigned flags = 0;
  const double ratio = epi.ctl->ratio;
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < epi.n; j += (int64_t)gridDim.x * blockDim.x) {
    if (xk_prev) {
      xk_prev[j] = epi.xk[j];
      xt_prev[j] = epi.xt[j];
    }
    const double cxj = epi.cx[j];
    const double xp = sub ? S_(cxj, aw[j]) : aw[j];
    if (!sub && !isfinite(xp)) flags |= kBadXPlus;
    epi.apply(j, xp, M_(S_(cxj, xp), ratio), red, flags);
  }
  __shared__ double sh[8][kRedX + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kRedX; ++k) red[k] = warp_sum(red[k]);
  flags = warp_or(flags);
  if (lane == 0) {
    for (int k = 0; k < kRedX; ++k) sh[warp][k] = red[k];
    sh[warp][kRedX] = (double)flags;
  }
  __syncthreads();
  if (threadIdx.x <= kRedX) {
    const int k = threadIdx.x;
    if (k < kRedX) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += sh[w][k];
      part[blockIdx.x * (kRedX + 1) + k] = s;
    } else {
      unsigned f = 0;
      for (int w = 0; w < 8; ++w) f |= (unsigned)sh[w][kRedX];
      part[blockIdx.x * (kRedX + 1) + kRedX] = (double)f;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) x_init_kernel(XEpi<T> epi, double* __restrict__ part) {
  double red[kRedX] = {};
  unsigned flags = 0;
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < epi.n; j += (int64_t)gridDim.x * blockDim.x)
    epi.apply(j, epi.xk[j], epi.xt[j], red, flags);
  __shared__ double sh[8][kRedX + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kRedX; ++k) red[k] = warp_sum(red[k]);
  flags = warp_or(flags);
  if (lane == 0) {
    for (int k = 0; k < kRedX; ++k) sh[warp][k] = red[k];
    sh[warp][kRedX] = (double)flags;
  }
  __syncthreads();
  if (threadIdx.x <= kRedX) {
    const int k = threadIdx.x;
    if (k < kRedX) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += sh[w][k];
      part[blockIdx.x * (kRedX + 1) + k] = s;
    } else {
      unsigned f = 0;
      for (int w = 0; w < 8; ++w) f |= (unsigned)sh[w][kRedX];
      part[blockIdx.x * (kRedX + 1) + kRedX] = (double)f;
    }
  }
}

// Z1 scalars: reduce the R partials -> red[2*ld .. 2*ld+8):
//   [r_pri^2, ||y||^2, f(y), drift_y^2, #bad y+, #bad y_1/2, f(y_full), f*(nu_full)]
__global__ void y_scalars_kernel(const double* __restrict__ rpart, int64_t count, double* __restrict__ out,
                                 const Ctl* ctl) {
  if (ctl->status != GF_STATUS_RUNNING) return;
  __shared__ double sh[256];
  __shared__ unsigned shf[256];
  for (int k = 0; k < kRedY; ++k) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) s += rpart[i * (kRedY + 1) + k];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[k < 4 ? k : k + 2] = sh[0];
    __syncthreads();
  }
  unsigned f = 0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) f |= (unsigned)rpart[i * (kRedY + 1) + kRedY];
  shf[threadIdx.x] = f;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int i = 0; i < 256; ++i) t |= shf[i];
    out[4] = (t & kBadYPlus) ? 1.0 : 0.0;
    out[5] = (t & kBadYHalf) ? 1.0 : 0.0;
  }
}

// Gap-based stopping at the full iterate (solver.py:205-218, :378-390):
// gap = ((f(y) + f*(nu)) + g(x)) + g*(mu) (problem.py:85); an infinite gap or
// objective never stops.
__device__ bool gap_test(Ctl* ctl, const Params& prm, const double* ys, const double* xs) {
  const double gap = A_(A_(A_(ys[6], ys[7]), xs[3]), xs[4]);
  ctl->gap = gap;
  ctl->gap_set = 1;
  if (!isfinite(gap)) return false;
  const double obj = A_(ys[6], xs[3]);
  if (!isfinite(obj)) return false;
  return gap <= A_(prm.abs_tol, M_(prm.rel_tol, fabs(obj)));
}

// Thread 0 of the last controller CTA, tall orientation: stop rule, degenerate
// checks, history row and adaptive rho of iteration k from the all-reduced y
// scalars ys, the x-side sums xs (+ flags word) and r_dual^2.
__device__ void decide_tall(Ctl* ctl, const Params& prm, const double* ys, const double* xs, double r2,
                            double* hist) {
  const int64_t k = ctl->k;
  const unsigned xf = (unsigned)xs[kRedX];
  const bool proj_bad = (xf & kBadXPlus) || ys[4] > 0.0;
  const bool prox_bad = (xf & kBadXHalf) || ys[5] > 0.0;
  if (k >= prm.max_iter) {  // past the last iteration: only its projection check remains
    ctl->iterations = prm.max_iter;
    if (proj_bad) { ctl->status = GF_STATUS_DEGENERATE; ctl->final_rho = ctl->rho_prev; }
    else { ctl->status = GF_STATUS_MAX_ITERATIONS; ctl->final_rho = ctl->rho; }
    return;
  }
  if (proj_bad || prox_bad) {   // solver.py:337-341 / :414-417 -> previous half iterate
    ctl->status = GF_STATUS_DEGENERATE;
    ctl->iterations = k;
    ctl->final_rho = proj_bad ? ctl->rho_prev : ctl->rho;
    return;
  }
  const double rho = ctl->rho;
  const double r_pri = sqrt(ys[0]);
  const double r_dual = sqrt(r2);
  const double eps_pri = prm.abs_tol + prm.rel_tol * sqrt(ys[1]);
  const double eps_dual = prm.abs_tol + prm.rel_tol * sqrt(xs[0]);
  const double obj = ys[2] + xs[1];
  double* hrow = hist + k * 8;
  hrow[0] = r_pri; hrow[1] = r_dual; hrow[2] = eps_pri; hrow[3] = eps_dual;
  hrow[4] = rho; hrow[5] = obj; hrow[6] = sqrt(ys[3] + xs[2]); hrow[7] = (double)ctl->inner;
  ctl->last_good = k;
  ctl->r_pri = r_pri; ctl->r_dual = r_dual; ctl->eps_pri = eps_pri; ctl->eps_dual = eps_dual;
  ctl->objective = obj;
  if ((r_pri <= eps_pri && r_dual <= eps_dual)       // solver.py:201, :373-376
      || (prm.gap && gap_test(ctl, prm, ys, xs))) {   // solver.py:378-390
    ctl->status = GF_STATUS_SOLVED;
    ctl->iterations = k + 1;
    ctl->final_rho = rho;
    return;
  }
  double nrho = rho, ratio = 1.0;                  // adapt_rho, solver.py:221-239
  if (prm.adaptive) {
    if (r_dual < eps_dual && prm.tau * (double)k > (double)ctl->l_mark) {
      nrho = prm.delta * rho;
      ratio = rho / nrho;
      ctl->u_mark = k;
    } else if (r_pri < eps_pri && prm.tau * (double)k > (double)ctl->u_mark) {
      nrho = rho / prm.delta;
      ratio = rho / nrho;
      ctl->l_mark = k;
    }
  }
  ctl->rho_prev = rho;
  ctl->rho = nrho;
  ctl->ratio = ratio;
  ctl->k = k + 1;
}

// Z step of a wide iteration (m < n): per column the x+ finiteness check and
// the r_dual terms, then the controller in the last CTA (tall iterations use
// zslab_tall_kernel).  red = [A_hat' w | A_hat' nu^ | y scalars];
// x+ = c_x - A_hat' w (projection.py:124-126); the y+ flags come from the
// G^-1 pass (spart).
__global__ void __launch_bounds__(256)
control_wide_kernel(Ctl* __restrict__ ctl, Params prm, const double* __restrict__ red, int64_t ld, int64_t n,
                    const double* __restrict__ cx, const double* __restrict__ e, const double* __restrict__ muh2,
                    double* __restrict__ zpart, const double* __restrict__ xpart, int64_t nxpart,
                    double* __restrict__ hist, const double* __restrict__ spart, int64_t nspart) {
  if (ctl->status != GF_STATUS_RUNNING) return;
  const int64_t k = ctl->k;
  const double* muh = muh2 + (k & 1) * n;
  double rd2 = 0.0;
  unsigned zflag = 0;
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double s1 = red[j], s2 = red[ld + j];
    if (!isfinite(S_(cx[j], s1))) zflag |= kBadXPlus;
    const double ej = e[j];
    const double rdj = A_(D_(s2, ej), D_(muh[j], ej)); // A' nu + mu in original space
    rd2 += rdj * rdj;
  }
  __shared__ double sh[256];
  __shared__ bool last;
  sh[threadIdx.x] = rd2;
  zflag = warp_or(zflag);
  if ((threadIdx.x & 31) == 0 && zflag) atomicOr((unsigned*)&ctl->zflags, zflag);
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    zpart[blockIdx.x] = sh[0];
    __threadfence();
    const unsigned t = atomicAdd(&ctl->ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // ---- last CTA: x-side partials of S(k-1) / x-init ----
  double xs[kRedX + 1];
  for (int q = 0; q < kRedX; ++q) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < nxpart; i += blockDim.x) s += xpart[i * (kRedX + 1) + q];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
      __syncthreads();
    }
    xs[q] = sh[0];
    __syncthreads();
  }
  {
    unsigned f = 0;
    for (int64_t i = threadIdx.x; i < nxpart; i += blockDim.x) f |= (unsigned)xpart[i * (kRedX + 1) + kRedX];
    sh[threadIdx.x] = (double)f;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned t = 0;
      for (int i = 0; i < 256; ++i) t |= (unsigned)sh[i];
      xs[kRedX] = (double)t;
    }
    __syncthreads();
  }
  unsigned sflag = 0;   // y+ = c_y + w flags of the Ginv pass
  {
    unsigned f = 0;
    for (int64_t i = threadIdx.x; i < nspart; i += blockDim.x) f |= (unsigned)spart[i];
    sh[threadIdx.x] = (double)f;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < 256; ++i) sflag |= (unsigned)sh[i];
  }
  if (threadIdx.x != 0) return;
  double r2 = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) r2 += zpart[b];
  ctl->ticket = 0;
  const unsigned zf = ctl->zflags;
  ctl->zflags = 0;
  const double* ys = red + 2 * ld;
  const unsigned xf = (unsigned)xs[kRedX];
  {
    // order of solver.py: prox checks (:337), residual stop (:373), then the
    // projection check (:414), then adapt_rho (:423)
    const bool prox_bad = (xf & kBadXHalf) || ys[5] > 0.0;
    const bool proj_bad = (zf & kBadXPlus) || (sflag & kBadYPlus);
    if (prox_bad) {
      ctl->status = GF_STATUS_DEGENERATE;
      ctl->iterations = k;
      ctl->final_rho = ctl->rho;
      return;
    }
    const double rho = ctl->rho;
    const double r_pri = sqrt(ys[0]);
    const double r_dual = sqrt(r2);
    const double eps_pri = prm.abs_tol + prm.rel_tol * sqrt(ys[1]);
    const double eps_dual = prm.abs_tol + prm.rel_tol * sqrt(xs[0]);
    const double obj = ys[2] + xs[1];
    double* hrow = hist + k * 8;
    hrow[0] = r_pri; hrow[1] = r_dual; hrow[2] = eps_pri; hrow[3] = eps_dual;
    hrow[4] = rho; hrow[5] = obj; hrow[6] = sqrt(ys[3] + xs[2]); hrow[7] = (double)ctl->inner;
    ctl->last_good = k;
    ctl->r_pri = r_pri; ctl->r_dual = r_dual; ctl->eps_pri = eps_pri; ctl->eps_dual = eps_dual;
    ctl->objective = obj;
    if ((r_pri <= eps_pri && r_dual <= eps_dual) || (prm.gap && gap_test(ctl, prm, ys, xs))) {
      ctl->status = GF_STATUS_SOLVED;
      ctl->iterations = k + 1;
      ctl->final_rho = rho;
      return;
    }
    if (proj_bad) {
      ctl->status = GF_STATUS_DEGENERATE;
      ctl->iterations = k + 1;
      ctl->final_rho = rho;
      return;
    }
    double nrho = rho, ratio = 1.0;
    if (prm.adaptive) {
      if (r_dual < eps_dual && prm.tau * (double)k > (double)ctl->l_mark) {
        nrho = prm.delta * rho;
        ratio = rho / nrho;
        ctl->u_mark = k;
      } else if (r_pri < eps_pri && prm.tau * (double)k > (double)ctl->u_mark) {
        nrho = rho / prm.delta;
        ratio = rho / nrho;
        ctl->l_mark = k;
      }
    }
    ctl->rho_prev = rho;
    ctl->rho = nrho;
    ctl->ratio = ratio;
    if (k + 1 >= prm.max_iter) {
      ctl->status = GF_STATUS_MAX_ITERATIONS;
      ctl->iterations = prm.max_iter;
      ctl->final_rho = nrho;
      return;
    }
    ctl->k = k + 1;
  }
}

// Z(k) in one launch for tall problems without a communicator: the column
// slab reduce, the y-scalar reduce and the controller (replaces colreduce +
// y_scalars + control_kernel).  CTA b owns columns [32 b, 32 b + 32): warp w
// sums slabs w, w + 8, ... of both column partials (fixed order, coalesced
// 256-byte rows), the 8 warp partials are added in warp order, then lane j of
// warp 0 forms rhs_j = c_x + A_hat' c_y and the r_dual term of its column.
// The last CTA (ticket) reduces the y records (rpart), the x records (xpart)
// and the per-CTA r_dual partials, all in fixed order, and runs the
// controller.  Deterministic: same sums in the same order on every run.
template <int K>
__device__ void block_sum_records(const double* __restrict__ rec, int64_t count, double (&out)[K + 1],
                                  double (*sh)[K + 1]) {
  // rec: count records of K sums + 1 flags word; out: the K sums + OR of flags
  double v[K + 1];
#pragma unroll
  for (int q = 0; q <= K; ++q) v[q] = 0.0;
  unsigned fl = 0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
#pragma unroll
    for (int q = 0; q < K; ++q) v[q] += rec[i * (K + 1) + q];
    fl |= (unsigned)rec[i * (K + 1) + K];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < K; ++q) v[q] = warp_sum(v[q]);
  fl = warp_or(fl);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < K; ++q) sh[warp][q] = v[q];
    sh[warp][K] = (double)fl;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += sh[w][q];
      out[q] = t;
    }
    unsigned f = 0;
    for (int w = 0; w < nw; ++w) f |= (unsigned)sh[w][K];
    out[K] = (double)f;
  }
  __syncthreads();
}

// Column sums of the slab partials for columns [c0, c0 + 32): warp w adds
// slabs w, w + 8, ...; the 8 warp partials are added in warp order.  Result
// in lane j of warp 0 (s1, s2).  Every CTA thread must call it.
__device__ __forceinline__ void slab_columns(const double* __restrict__ cpart, int64_t slabs, int64_t ld, int64_t n,
                                             int64_t c0, double (*part)[2][33], double& s1, double& s2) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = c0 + lane;
  s1 = 0.0;
  s2 = 0.0;
  if (j < n) {   // four independent chains: 8 loads in flight per lane
    double a1[4] = {0.0, 0.0, 0.0, 0.0}, a2[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t sl = warp;
    for (; sl + 24 < slabs; sl += 32)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a1[u] += cpart[(2 * (sl + 8 * u)) * ld + j];
        a2[u] += cpart[(2 * (sl + 8 * u) + 1) * ld + j];
      }
    for (; sl < slabs; sl += 8) {   // remainder into chain 0 (static indices: no local memory)
      a1[0] += cpart[(2 * sl) * ld + j];
      a2[0] += cpart[(2 * sl + 1) * ld + j];
    }
    s1 = (a1[0] + a1[1]) + (a1[2] + a1[3]);
    s2 = (a2[0] + a2[1]) + (a2[2] + a2[3]);
  }
  part[warp][0][lane] = s1;
  part[warp][1][lane] = s2;
  __syncthreads();
  if (warp == 0) {
    s1 = part[0][0][lane];
    s2 = part[0][1][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) { s1 += part[w][0][lane]; s2 += part[w][1][lane]; }
  }
  __syncthreads();
}

// The y records in the controller's scalar layout (see y_scalars_kernel):
// [r_pri^2, ||y||^2, f(y), drift_y^2, bad y+, bad y_1/2, f(y_full), f*(nu_full)]
__device__ __forceinline__ void y_layout(const double (&yr)[kRedY + 1], double* ys) {
  const unsigned yf = (unsigned)yr[kRedY];
  ys[0] = yr[0]; ys[1] = yr[1]; ys[2] = yr[2]; ys[3] = yr[3];
  ys[4] = (yf & kBadYPlus) ? 1.0 : 0.0;
  ys[5] = (yf & kBadYHalf) ? 1.0 : 0.0;
  ys[6] = yr[4]; ys[7] = yr[5];
}

// Row-partitioned runs: the same reductions as zslab_tall_kernel<true>, in the
// same order, written to red = [A' c_y | A' nu^ | y scalars] for the
// all-reduce; zslab_tall_kernel<false> then reads them.  With one rank the
// result is bit-identical to the communicator-free path.
__global__ void __launch_bounds__(256)
zreduce_kernel(const Ctl* __restrict__ ctl, const double* __restrict__ cpart, int64_t slabs, int64_t ld, int64_t n,
               const double* __restrict__ rpart, int64_t nrpart, double* __restrict__ red) {
  if (ctl->status != GF_STATUS_RUNNING) return;
  __shared__ double part[8][2][33];
  __shared__ double shr[8][kRedY + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t c0 = (int64_t)blockIdx.x * 32; c0 < ld; c0 += (int64_t)gridDim.x * 32) {
    double s1, s2;
    slab_columns(cpart, slabs, ld, ld, c0, part, s1, s2);
    if (warp == 0 && c0 + lane < ld) {
      red[c0 + lane] = s1;
      red[ld + c0 + lane] = s2;
    }
  }
  if (blockIdx.x == 0) {
    double yr[kRedY + 1];
    block_sum_records<kRedY>(rpart, nrpart, yr, shr);
    if (threadIdx.x == 0) y_layout(yr, red + 2 * ld);
  }
}

template <typename T, bool FROM_SLABS>
__global__ void __launch_bounds__(256)
zslab_tall_kernel(Ctl* __restrict__ ctl, Params prm, const double* __restrict__ cpart, int64_t slabs, int64_t ld,
                  int64_t n, const double* __restrict__ rpart, int64_t nrpart, const double* __restrict__ cx,
                  const double* __restrict__ e, const double* __restrict__ muh2, T* __restrict__ rhs_T,
                  double* __restrict__ zpart, const double* __restrict__ xpart, int64_t nxpart,
                  double* __restrict__ hist, double* __restrict__ red) {
  pdl_wait();
  pdl_trigger();
  if (ctl->status != GF_STATUS_RUNNING) return;
  __shared__ double part[8][2][33];
  __shared__ double shr[8][kRedY + 1];
  __shared__ double shx[8][kRedX + 1];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t k = ctl->k;
  const double* muh = muh2 + (k & 1) * n;
  // the record reductions (x side; y side from slabs) do not wait for the
  // column sums: CTA 0 does them first, off the last CTA's critical path,
  // into red[2 ld + kScal ..] ([y scalars (kScal) | x sums + flags])
  double* recs = red + 2 * ld + kScal;
  if (blockIdx.x == 0) {
    double yr[kRedY + 1], xs0[kRedX + 1];
    if (FROM_SLABS) block_sum_records<kRedY>(rpart, nrpart, yr, shr);
    block_sum_records<kRedX>(xpart, nxpart, xs0, shx);
    if (threadIdx.x == 0) {
      if (FROM_SLABS) y_layout(yr, recs);
      for (int q = 0; q <= kRedX; ++q) recs[kScal + q] = xs0[q];
    }
  }
  double rd2 = 0.0;
  for (int64_t c0 = (int64_t)blockIdx.x * 32; c0 < n; c0 += (int64_t)gridDim.x * 32) {
    const int64_t j = c0 + lane;
    double s1 = 0.0, s2 = 0.0;
    if (FROM_SLABS) {
      slab_columns(cpart, slabs, ld, n, c0, part, s1, s2);
    } else if (j < n) {
      s1 = red[j];
      s2 = red[ld + j];
    }
    if (warp == 0 && j < n) {
      rhs_T[j] = (T)A_(cx[j], s1);                      // c + A_hat' d (projection.py:121)
      const double ej = e[j];
      const double rdj = A_(D_(s2, ej), D_(muh[j], ej));  // A' nu + mu in original space
      rd2 += rdj * rdj;
    }
  }
  if (warp == 0) {
    rd2 = warp_sum(rd2);
    if (lane == 0) {
      zpart[blockIdx.x] = rd2;
      __threadfence();
      last = atomicAdd(&ctl->ticket, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double zs[8];
  {
    double z = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) z += zpart[b];
    z = warp_sum(z);
    if (lane == 0) zs[warp] = z;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double r2 = 0.0;
  for (int w = 0; w < 8; ++w) r2 += zs[w];
  ctl->ticket = 0;
  double* ys = red + 2 * ld;
  if (FROM_SLABS)
    for (int q = 0; q < kScal; ++q) ys[q] = recs[q];
  double xs[kRedX + 1];
  for (int q = 0; q <= kRedX; ++q) xs[q] = recs[kScal + q];
  decide_tall(ctl, prm, ys, xs, r2, hist);
}

// --------------------------------------------- Z step in the fused pass --
// The fused schedules end with the Z step inside the same launch (ZTail, run
// by every thread of every CTA after the main loop; the pass is persistent:
// one CTA per SM, all co-resident, so a grid barrier is safe):
//   barrier -> CTA b sums the slabs of columns [n b / G, n (b+1) / G) in
//              fixed slab order; CTA 0 the y records
//   mode 2 (one GPU): rhs = c_x + A' c_y and the r_dual^2 partial of those
//              columns at once, CTA 0's x records, and the controller in the
//              last CTA to arrive (ticket) -- one barrier, no second launch
//   mode 1 (row partition): the column sums and y scalars go to red, which is
//              all-reduced; zfinish_kernel then finishes the same columns in
//              the same lane order with the same grid, so one rank is
//              bit-identical to the communicator-free path.
// This replaces the separate Z launch (slab sums + controller: ~20 us at
// 200000 x 5000, most of it launch ramp and the serial tail).
__device__ __forceinline__ void grid_sync(unsigned* cnt, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vg = gen;
    const unsigned g0 = *vg;
    __threadfence();
    if (atomicAdd(cnt, 1u) == gridDim.x - 1) {
      atomicExch(cnt, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vg == g0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

constexpr int kTailThreads = 256;   // threads of a CTA that do the Z work (fixed: same sums in both modes)
constexpr int kTailSlabs = 20;      // slab loads in flight per lane (per warp: slabs w, w + 8, ...)

template <typename T>
struct ZTail {
  Ctl* ctl;
  Params prm;
  const double* cpart;
  int64_t slabs, ld, n;
  const double* rpart;
  int64_t nrpart;
  const double* cx;
  const double* e;
  const double* muh2;
  T* rhs_T;
  double* zpart;
  const double* xpart;
  int64_t nxpart;
  double* hist;
  double* red;   // [2 ld column sums | kScal y scalars | kRedX + 1 x sums]
  int mode;      // 0 off, 1 column sums + y scalars only, 2 the whole Z step

  __device__ bool on() const { return mode != 0; }

  // Columns [n b / G, n (b+1) / G) of CTA b, 32 at a time: warp w < 8 loads
  // slabs w, w + 8, ... of both sums (all loads issued before the adds), a
  // fixed-order combine over the 8 warps in shared memory, then warp 0's lane
  // l holds column cc + l: mode 1 stores it in red, mode 2 finishes it.
  __device__ void run() const {
    grid_sync(&ctl->gcnt, &ctl->ggen);
    __shared__ double part[8][2][33];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool act = tid < kTailThreads;
    const int64_t G = gridDim.x, b = blockIdx.x;
    const int64_t c0 = n * b / G, c1 = n * (b + 1) / G;
    const double* muh = muh2 + (ctl->k & 1) * n;
    double rd2 = 0.0;
    for (int64_t cc = c0; cc < c1; cc += 32) {   // uniform trip count in the CTA
      const int64_t j = cc + lane;
      double s1 = 0.0, s2 = 0.0;
      if (act && j < c1) {
        for (int64_t sb = warp; sb < slabs; sb += 8 * kTailSlabs) {
          double v1[kTailSlabs], v2[kTailSlabs];
#pragma unroll
          for (int u = 0; u < kTailSlabs; ++u) {
            const int64_t sl = sb + 8 * u;
            v1[u] = sl < slabs ? cpart[(2 * sl) * ld + j] : 0.0;
            v2[u] = sl < slabs ? cpart[(2 * sl + 1) * ld + j] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < kTailSlabs; ++u) { s1 += v1[u]; s2 += v2[u]; }
        }
      }
      if (act) {
        part[warp][0][lane] = s1;
        part[warp][1][lane] = s2;
      }
      __syncthreads();
      if (warp == 0 && j < c1) {
        double t1 = part[0][0][lane], t2 = part[0][1][lane];
#pragma unroll
        for (int w = 1; w < 8; ++w) { t1 += part[w][0][lane]; t2 += part[w][1][lane]; }
        if (mode == 1) {
          red[j] = t1;
          red[ld + j] = t2;
        } else {
          rd2 += column(j, t1, t2, muh);
        }
      }
      __syncthreads();
    }
    if (b == 0) y_records();
    if (mode == 2) close(rd2);
  }

  // rhs_j = c_x,j + (A_hat' c_y)_j (projection.py:121); returns the r_dual
  // term ((A' nu + mu)_j in the original space)^2
  __device__ double column(int64_t j, double s1, double s2, const double* muh) const {
    rhs_T[j] = (T)A_(cx[j], s1);
    const double ej = e[j];
    const double rdj = A_(D_(s2, ej), D_(muh[j], ej));
    return rdj * rdj;
  }

  // y records (rpart) -> the controller's scalar layout at red + 2 ld
  __device__ void y_records() const {
    __shared__ double shr[8][kRedY + 1];
    double yr[kRedY + 1];
    block_records<kRedY>(rpart, nrpart, yr, shr);
    if (threadIdx.x == 0) y_layout(yr, red + 2 * ld);
  }

  // fixed-order sums of `count` records of K values + a flags word, over the
  // first kTailThreads threads; thread 0 gets the result
  template <int K>
  __device__ void block_records(const double* rec, int64_t count, double (&out)[K + 1], double (*sh)[K + 1]) const {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool act = tid < kTailThreads;
    double v[K + 1];
#pragma unroll
    for (int q = 0; q <= K; ++q) v[q] = 0.0;
    unsigned fl = 0;
    if (act)
      for (int64_t i = tid; i < count; i += kTailThreads) {
#pragma unroll
        for (int q = 0; q < K; ++q) v[q] += rec[i * (K + 1) + q];
        fl |= (unsigned)rec[i * (K + 1) + K];
      }
#pragma unroll
    for (int q = 0; q < K; ++q) v[q] = warp_sum(v[q]);
    fl = warp_or(fl);
    if (act && lane == 0) {
#pragma unroll
      for (int q = 0; q < K; ++q) sh[warp][q] = v[q];
      sh[warp][K] = (double)fl;
    }
    __syncthreads();
    if (tid == 0) {
      unsigned f = 0;
      for (int q = 0; q < K; ++q) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += sh[w][q];
        out[q] = t;
      }
      for (int w = 0; w < 8; ++w) f |= (unsigned)sh[w][K];
      out[K] = (double)f;
    }
    __syncthreads();
  }

  // this CTA's r_dual^2 partial (held by warp 0's lanes), CTA 0's x records,
  // then the controller in the last CTA to arrive
  __device__ void close(double rd2) const {
    __shared__ double shx[8][kRedX + 1];
    __shared__ bool last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t G = gridDim.x, b = blockIdx.x;
    double* xs = red + 2 * ld + kScal;
    if (b == 0) {
      double xr[kRedX + 1];
      block_records<kRedX>(xpart, nxpart, xr, shx);
      if (tid == 0)
        for (int q = 0; q <= kRedX; ++q) xs[q] = xr[q];
    }
    if (warp == 0) {
      rd2 = warp_sum(rd2);
      if (lane == 0) {
        zpart[b] = rd2;
        __threadfence();
        last = atomicAdd(&ctl->ticket, 1u) == (unsigned)G - 1;
      }
    }
    __syncthreads();
    if (!last || warp != 0) return;
    __threadfence();
    double z = 0.0;   // fixed order: lane l sums CTAs l, l + 32, ...; then a fixed tree
    for (int64_t i = lane; i < G; i += 32) z += ((volatile const double*)zpart)[i];
    z = warp_sum(z);
    if (lane != 0) return;
    ctl->ticket = 0;
    decide_tall(ctl, prm, red + 2 * ld, xs, z, hist);
  }

  // mode 1's second half, after the all-reduce of red: the same columns in
  // the same lane order as run()'s mode 2, then close()
  __device__ void finish() const {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t G = gridDim.x, b = blockIdx.x;
    const int64_t c0 = n * b / G, c1 = n * (b + 1) / G;
    const double* muh = muh2 + (ctl->k & 1) * n;
    double rd2 = 0.0;
    if (warp == 0)
      for (int64_t cc = c0; cc < c1; cc += 32) {
        const int64_t j = cc + lane;
        if (j < c1) rd2 += column(j, red[j], red[ld + j], muh);
      }
    (void)tid;
    close(rd2);
  }
};

// Row-partitioned fused schedules: finish() after the all-reduce of red, with
// the fused pass's grid (same column partition: one rank is bit-identical to
// the single-GPU in-kernel Z step).
template <typename T>
__global__ void __launch_bounds__(kTailThreads) zfinish_kernel(ZTail<T> z) {
  pdl_trigger();   // the next iteration's G^-1 ring may start its constant-matrix prefetch
  if (z.ctl->status != GF_STATUS_RUNNING) return;
  z.finish();
}

// ------------------------------------------------------------- results --
__global__ void result_kernel(const Ctl* ctl, int64_t n, int64_t m, const double* __restrict__ xh2,
                              const double* __restrict__ muh2, const double* __restrict__ yh2,
                              const double* __restrict__ nuh2, const double* __restrict__ e,
                              const double* __restrict__ d, double* x, double* mu, double* y, double* nu) {
  const int64_t L = ctl->last_good;
  const int64_t bx = (L & 1) * n, by = (L & 1) * m;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < n; j += stride) {
    x[j] = L < 0 ? 0.0 : xh2[bx + j];
    mu[j] = L < 0 ? 0.0 : muh2[bx + j] / e[j];       // unscale (solver.py:188)
  }
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < m; i += stride) {
    y[i] = L < 0 ? 0.0 : yh2[by + i];
    nu[i] = L < 0 ? 0.0 : d[i] * nuh2[by + i];
  }
}

__global__ void snapshot_kernel(const Ctl* ctl, int64_t n, int64_t m, const double* xh2, const double* yh2,
                                const double* e, const double* d, double* xhh, double* yhh) {
  const int64_t L = ctl->last_good < 0 ? 0 : ctl->last_good;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < n; j += stride) xhh[j] = xh2[(L & 1) * n + j] / e[j];
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < m; i += stride) yhh[i] = yh2[(L & 1) * m + i] * d[i];
}

__global__ void warm_init_kernel(const double* __restrict__ x0, const double* __restrict__ nu0, const double* e,
                                 const double* d, int64_t n, int64_t m, double rho, double* xk, double* nuhat0,
                                 double* yt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < n; j += stride)
    xk[j] = x0 ? x0[j] / e[j] : 0.0;                 // solver.py:301
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < m; i += stride) {
    if (nu0) {
      const double nh = nu0[i] / d[i];               // solver.py:304-305
      nuhat0[i] = nh;
      yt[i] = -nh / rho;
    } else {
      yt[i] = 0.0;
    }
  }
}

__global__ void div_into(const double* __restrict__ src, int64_t n, double rho, double* __restrict__ dst) {
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    dst[j] = src[j] / rho;                           // solver.py:306
}

}  // namespace gf

// Pinned controller read-back buffers (2 x Ctl per solver) come from a
// process-wide free list: cudaMallocHost / cudaFreeHost per solver cost
// milliseconds and synchronise the device.
namespace gf {
static std::mutex g_pinned_mu;
static std::vector<Ctl*> g_pinned_free;
static Ctl* pinned_acquire() {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (!g_pinned_free.empty()) {
      Ctl* p = g_pinned_free.back();
      g_pinned_free.pop_back();
      return p;
    }
  }
  Ctl* p = nullptr;
  GF_CUDA(cudaMallocHost(&p, 2 * sizeof(Ctl)));
  return p;
}
static void pinned_release(Ctl* p) {
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_pinned_free.push_back(p);
}
}  // namespace gf

// ============================================================== driver ====
using namespace gf;

struct gf_solver {
  gf_setup* S = nullptr;
  int dtype = GF_F64;
  int64_t m = 0, n = 0, ld = 0, q = 0, ldq = 0;
  bool tall = true;
  bool indirect = false;   // CGLS projection (projection.py:130-162)
  double ptol = -1.0;      // fixed CGLS tolerance, <= 0: schedule
  DBuf ypl, wv, spart;   // wide: y+ of the last projection, w, Ginv-pass flags
  DBuf xkp, xtp;         // wide: x^, x~ of the last recorded iteration (trace snapshots)
  DBuf xplus;            // indirect: CGLS iterate / x+
  Params prm{};
  TermsDev f, g;
  DBuf ctl, hist;
  DBuf xk, xt, cx, xh2, muh2, yk, yt, cy, yh2, nuh2;
  DBuf xk_T, xh_T, rhs_T;
  DBuf rpart, cpart, red, zpart, xpart;
  int64_t grid_r = 1, grid_s = 1, grid_z = 1, grid_zt = 1;
  ColPlan cplan;
  FusedPlan fplan;
  FusedPlan2 fplan2;  // two-CTA cluster variant (rows of 40 KB and more)
  RingPlan rplan;     // S step on the TMA row ring (tall, direct)
  SymPlan splan;      // S step on the lower triangle of G^-1 (tall, direct; preferred)
  CUtensorMap sym_tm; // 64 x 64 tiles of G^-1
  DBuf sympart;       // per-tile row / column partials of the S step
  int warm_x = 0;
  int64_t next_step = 0;  // step k = [S(k-1)], R(k), C(k), Z(k)
  Ctl host{};
  Ctl* pinned = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  cudaEvent_t ev_done[2] = {nullptr, nullptr};   // controller snapshots of in-flight chunks
  double elapsed_ms = 0.0;
  int64_t launches = 0;  // kernels launched by solver_run
  int64_t inner_host = 0;  // H2D source of the last CGLS count (wide indirect)
  // optional per-kernel timing (gf_solver_profile): events around each launch
  bool profile = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> ev_marks;  // (kernel class, pool index of start event)
  double kms[8] = {0};
  int64_t kcount[8] = {0};
  ~gf_solver() {
    if (pinned) pinned_release(pinned);
    if (ev_a) cudaEventDestroy(ev_a);
    if (ev_b) cudaEventDestroy(ev_b);
    for (auto e : ev_done)
      if (e) cudaEventDestroy(e);
    for (auto e : ev_pool) cudaEventDestroy(e);
  }
  // Kernel classes: 0 S (Ginv GEMV + x side), 1 R (row pass + y side),
  // 2 C (column pass), 3 column-slab reduce, 4 y scalars, 5 controller,
  // 6 NCCL all-reduce, 7 fused row+column pass (replaces 1 and 2).
  void mark(int cls, cudaStream_t st, bool begin) {
    if (!profile) return;
    const size_t idx = ev_marks.size() * 2 + (begin ? 0 : 1);
    while (ev_pool.size() <= idx) {
      cudaEvent_t e;
      GF_CUDA(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    GF_CUDA(cudaEventRecord(ev_pool[idx], st));
    if (!begin) ev_marks.emplace_back(cls, (int)(idx - 1));
  }
  void collect() {
    for (auto& mk : ev_marks) {
      float ms = 0.f;
      GF_CUDA(cudaEventElapsedTime(&ms, ev_pool[mk.second], ev_pool[mk.second + 1]));
      kms[mk.first] += ms;
      kcount[mk.first] += 1;
    }
    ev_marks.clear();
  }
};

namespace gf {

template <typename T>
static YEpi<T> make_yepi(gf_solver* s) {
  YEpi<T> y;
  y.ctl = s->ctl.as<Ctl>();
  y.f = s->f.view;
  y.d = s->S->d.as<double>();
  y.yk = s->yk.as<double>(); y.yt = s->yt.as<double>(); y.cy = s->cy.as<double>();
  y.yh2 = s->yh2.as<double>(); y.nuh2 = s->nuh2.as<double>();
  y.m = s->m; y.alpha = s->prm.alpha; y.warm_x = s->warm_x; y.gap = s->prm.gap;
  return y;
}

// Launch with the programmatic-stream-serialization attribute when `pdl`
// (the three kernels of a tall iteration: each waits on its predecessor with
// pdl_wait(), so launch processing and the fused kernel's first ring fill
// overlap the previous kernel's tail).
template <typename... KArgs, typename... Args>
static void launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  GF_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

static bool use_pdl(const gf_solver* s) {
  static const bool off = [] {
    const char* e = getenv("GF_DISABLE_PDL");
    return e && e[0] == '1';
  }();
  // (under a communicator too: the launches that carry the attribute -- the
  // G^-1 ring and the fused pass -- follow one of this library's kernels;
  // the kernels after the NCCL all-reduce are launched without it)
  return !off && !s->profile;
}

// attr_only: set the dynamic shared-memory limit of the instance (at create)
// The Z step carried by the fused pass: mode 2 on one GPU (whole step in
// the launch), mode 1 under a communicator (column sums + y scalars; the
// all-reduce and zfinish_kernel follow).
template <typename T>
static ZTail<T> make_ztail(gf_solver* s, int64_t slabs, int64_t nrpart) {
  ZTail<T> z;
  z.ctl = s->ctl.as<Ctl>();
  z.prm = s->prm;
  z.cpart = s->cpart.as<double>();
  z.slabs = slabs;
  z.ld = s->ld;
  z.n = s->n;
  z.rpart = s->rpart.as<double>();
  z.nrpart = nrpart;
  z.cx = s->cx.as<double>();
  z.e = s->S->e.as<double>();
  z.muh2 = s->muh2.as<double>();
  z.rhs_T = s->rhs_T.as<T>();
  z.zpart = s->zpart.as<double>();
  z.xpart = s->xpart.as<double>();
  z.nxpart = s->grid_s;
  z.hist = s->hist.as<double>();
  z.red = s->red.as<double>();
  z.mode = comm_active(s->S->comm) ? 1 : 2;
  return z;
}

template <typename T, int NV, int TR, int CW>
static void fused_go(gf_solver* s, cudaStream_t st, bool attr_only) {
  const FusedPlan& p = s->fplan;
  auto kern = fused_rowcol_kernel<T, NV, TR, CW, YEpi<T>, ZTail<T>>;
  if (attr_only) {
    GF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    return;
  }
  launch_k(use_pdl(s), kern, dim3(p.grid), dim3(fused_threads(CW)), p.smem, st, (const T*)s->S->A->data, s->m,
           s->ld, (const T*)s->xk_T.as<T>(), (const T*)s->xh_T.as<T>(), make_yepi<T>(s), p.nslot,
           s->rpart.as<double>(), s->cpart.as<double>(), make_ztail<T>(s, p.grid, (int64_t)p.ne * p.grid));
  GF_CHECK_LAUNCH();
}

template <typename T, int NV, int CW>
static void fused_tr(gf_solver* s, cudaStream_t st, bool attr_only) {
  switch (s->fplan.tr) {
    case 4: fused_go<T, NV, 4, CW>(s, st, attr_only); break;
    case 2: fused_go<T, NV, 2, CW>(s, st, attr_only); break;
    default: fused_go<T, NV, 1, CW>(s, st, attr_only); break;
  }
}

// plan_fused: CW = 8 for NV <= 5; 12 when 8 would need more (NV in {4, 5});
// 16 and 20 for NV = 4; 20 with NV 5 or 6 for the widest fused rows
template <typename T>
static void fused_dispatch(gf_solver* s, cudaStream_t st, bool attr_only) {
  const int nv = s->fplan.nv;
  switch (s->fplan.cw) {
    case 8:
      switch (nv) {
        case 1: fused_tr<T, 1, 8>(s, st, attr_only); break;
        case 2: fused_tr<T, 2, 8>(s, st, attr_only); break;
        case 3: fused_tr<T, 3, 8>(s, st, attr_only); break;
        case 4: fused_tr<T, 4, 8>(s, st, attr_only); break;
        default: fused_tr<T, 5, 8>(s, st, attr_only); break;
      }
      return;
    case 12:
      if (nv == 4) fused_tr<T, 4, 12>(s, st, attr_only); else fused_tr<T, 5, 12>(s, st, attr_only);
      return;
    case 16:
      fused_tr<T, 4, 16>(s, st, attr_only);
      return;
    default:
      switch (nv) {
        case 4: fused_tr<T, 4, 20>(s, st, attr_only); break;
        case 5: fused_tr<T, 5, 20>(s, st, attr_only); break;
        default: fused_tr<T, 6, 20>(s, st, attr_only); break;
      }
      return;
  }
}

// Two-CTA cluster variant.  attr_only: set the shared-memory limit and
// return the number of co-resident clusters of this instance.
template <typename T, int NV, int TR, int CW, int CL, int LAG = 0>
static int fused2_go(gf_solver* s, cudaStream_t st, bool attr_only) {
  const FusedPlan2& p = s->fplan2;
  auto kern = fused_rowcol_cl_kernel<T, NV, TR, CW, CL, YEpi<T>, ZTail<T>, LAG>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(attr_only ? CL * (num_sms() / CL) : p.grid));
  cfg.blockDim = dim3(fused_threads_lag(CW, LAG));
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  if (attr_only) {
    GF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    if (CL > 8) GF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cfg.numAttrs = 1;
    int ncl = 0;
    GF_CUDA(cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &cfg));
    return ncl;
  }
  cfg.numAttrs = use_pdl(s) ? 2 : 1;
  GF_CUDA(cudaLaunchKernelEx(&cfg, kern, (const T*)s->S->A->data, s->m, s->ld, (const T*)s->xk_T.as<T>(),
                             (const T*)s->xh_T.as<T>(), make_yepi<T>(s), p.nslot, p.hvec, s->rpart.as<double>(),
                             s->cpart.as<double>(), make_ztail<T>(s, p.grid / CL, (int64_t)p.ne * p.grid),
                             p.nslotc));
  GF_CHECK_LAUNCH();
  return 0;
}

template <typename T, int NV, int CW, int CL>
static int fused2_tr(gf_solver* s, cudaStream_t st, bool attr_only) {
  return s->fplan2.tr >= 2 ? fused2_go<T, NV, 2, CW, CL>(s, st, attr_only) : fused2_go<T, NV, 1, CW, CL>(s, st, attr_only);
}

// cluster pass: the 2-CTA instances cover the compute-warp shapes of
// plan_fused; 4-, 8- and 9-CTA clusters (rows of 80 / 160 KB: fp64 n = 10000
// / 20000) the 8-warp ones
template <typename T, int CL>
static int fused2_cw(gf_solver* s, cudaStream_t st, bool attr_only) {
  const int nv = s->fplan2.nv;
  if constexpr (CL > 2) {
    switch (nv) {
      case 1: case 2: case 3: return fused2_tr<T, 3, 8, CL>(s, st, attr_only);
      case 4: return fused2_tr<T, 4, 8, CL>(s, st, attr_only);
      default: return fused2_tr<T, 5, 8, CL>(s, st, attr_only);
    }
  } else {
    switch (s->fplan2.cw) {
      case 8:
        switch (nv) {
          case 1: case 2: case 3: return fused2_tr<T, 3, 8, 2>(s, st, attr_only);
          case 4: return fused2_tr<T, 4, 8, 2>(s, st, attr_only);
          default: return fused2_tr<T, 5, 8, 2>(s, st, attr_only);
        }
      case 12:
        return nv == 4 ? fused2_tr<T, 4, 12, 2>(s, st, attr_only) : fused2_tr<T, 5, 12, 2>(s, st, attr_only);
      case 16:
        return fused2_tr<T, 4, 16, 2>(s, st, attr_only);
      default:
        switch (nv) {
          case 4: return fused2_tr<T, 4, 20, 2>(s, st, attr_only);
          case 5: return fused2_tr<T, 5, 20, 2>(s, st, attr_only);
          default: return fused2_tr<T, 6, 20, 2>(s, st, attr_only);
        }
    }
  }
}

// Lagged cluster pass for Newton-prox losses (gf_fused.cuh, LAG): 2-CTA
// clusters of 8 compute warps, two rows per group.  C2 (fp32 logistic
// 100000 x 10000) per pass: lag 4 0.950 ms, 6 0.892, 8 0.885, 12 0.907,
// 16 1.11 (the re-read rows no longer stay in L2).
constexpr int kNewtonLag = 8;

template <typename T>
static int fused2_dispatch(gf_solver* s, cudaStream_t st, bool attr_only) {
  if (s->fplan2.lag > 0) {
    switch (s->fplan2.nv) {
      case 1: case 2: case 3: return fused2_go<T, 3, 2, 8, 2, kNewtonLag>(s, st, attr_only);
      case 4: return fused2_go<T, 4, 2, 8, 2, kNewtonLag>(s, st, attr_only);
      default: return fused2_go<T, 5, 2, 8, 2, kNewtonLag>(s, st, attr_only);
    }
  }
  switch (s->fplan2.cl) {
    case 9: return fused2_cw<T, 9>(s, st, attr_only);
    case 8: return fused2_cw<T, 8>(s, st, attr_only);
    case 4: return fused2_cw<T, 4>(s, st, attr_only);
    default: return fused2_cw<T, 2>(s, st, attr_only);
  }
}

template <typename T>
static XEpi<T> make_xepi(gf_solver* s);

template <typename T, int NV, int CW>
static void ring_go(gf_solver* s, cudaStream_t st, bool attr_only) {
  const RingPlan& p = s->rplan;
  auto kern = ring_gemv_kernel<T, NV, CW, XEpi<T>>;
  if (attr_only) {
    GF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    return;
  }
  launch_k(use_pdl(s), kern, dim3(p.grid), dim3((CW + 2) * 32), p.smem, st, (const T*)s->S->P->ginv.as<T>(), s->q,
           s->ldq, (const T*)s->rhs_T.as<T>(), make_xepi<T>(s), p.nslot, s->xpart.as<double>(), s->grid_s);
}

template <typename T>
static void sym_go(gf_solver* s, cudaStream_t st, bool attr_only) {
  const SymPlan& p = s->splan;
  auto kern = sym_gemv_kernel<T, XEpi<T>>;
  if (attr_only) {
    GF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    return;
  }
  launch_k(use_pdl(s), kern, dim3(p.grid), dim3(sym_threads<T>()), p.smem, st, s->sym_tm, s->q,
           (const T*)s->rhs_T.as<T>(), make_xepi<T>(s), p.nslot, p.nb, p.nt, s->sympart.as<double>(),
           &s->ctl.as<Ctl>()->scnt, &s->ctl.as<Ctl>()->sgen, s->xpart.as<double>(), s->grid_s);
}

// 2-D tensor map over G^-1 (q columns x q rows, row stride ldq): 64 x 64
// boxes, zero fill past q in both directions.  The driver entry point comes
// through the runtime (no libcuda link dependency).
static CUtensorMap sym_map(const void* g, int64_t q, int64_t ldq, int dtype) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    GF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
    GF_REQUIRE(fn != nullptr && qr == cudaDriverEntryPointSuccess, GF_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const size_t es = dtype == GF_F32 ? 4 : 8;
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)q, (cuuint64_t)q};
  const cuuint64_t strides[1] = {(cuuint64_t)(ldq * es)};
  const cuuint32_t box[2] = {(cuuint32_t)kSymTB, (cuuint32_t)kSymTB};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&m, dtype == GF_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                            const_cast<void*>(g), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  GF_REQUIRE(r == CUDA_SUCCESS, GF_E_CUDA, "cuTensorMapEncodeTiled (G^-1 tiles) failed");
  return m;
}

template <typename T>
static void ring_dispatch(gf_solver* s, cudaStream_t st, bool attr_only) {
  const int nv = s->rplan.nv;
  switch (s->rplan.cw) {
    case 8:
      switch (nv) {
        case 1: ring_go<T, 1, 8>(s, st, attr_only); break;
        case 2: ring_go<T, 2, 8>(s, st, attr_only); break;
        case 3: ring_go<T, 3, 8>(s, st, attr_only); break;
        case 4: ring_go<T, 4, 8>(s, st, attr_only); break;
        default: ring_go<T, 5, 8>(s, st, attr_only); break;
      }
      return;
    case 12:
      if (nv == 4) ring_go<T, 4, 12>(s, st, attr_only); else ring_go<T, 5, 12>(s, st, attr_only);
      return;
    case 16:
      ring_go<T, 4, 16>(s, st, attr_only);
      return;
    default:
      ring_go<T, 4, 20>(s, st, attr_only);
      return;
  }
}

template <typename T>
static void fused_prepare(gf_solver* s) { fused_dispatch<T>(s, nullptr, true); }

template <typename T>
static void launch_fused(gf_solver* s, cudaStream_t st) { fused_dispatch<T>(s, st, false); }

template <typename T>
static XEpi<T> make_xepi(gf_solver* s) {
  XEpi<T> x;
  x.ctl = s->ctl.as<Ctl>();
  x.g = s->g.view;
  x.e = s->S->e.as<double>();
  x.xk = s->xk.as<double>(); x.xt = s->xt.as<double>(); x.cx = s->cx.as<double>();
  x.xh2 = s->xh2.as<double>(); x.muh2 = s->muh2.as<double>();
  x.xk_T = s->xk_T.as<T>(); x.xh_T = s->xh_T.as<T>();
  x.n = s->n; x.alpha = s->prm.alpha; x.wide = s->tall ? 0 : 1; x.gap = s->prm.gap;
  return x;
}

// G^-1 GEMV grid: one wave of resident CTAs (the register count of the XEpi
// instance allows 2 per SM), rows spread evenly over the warps.
template <typename T>
static int64_t ginv_grid(int64_t q, int sms) {
  int b = 0;
  GF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rowgemv_kernel<T, 1, XEpi<T>>, kRowThreads, 0));
  return std::max<int64_t>(1, std::min<int64_t>(ceil_div(q, kRowWarps), (int64_t)sms * std::max(b, 1)));
}

// GF_LAUNCH_SYNC=1 (debug): synchronise after every iteration kernel and log it
static void dbg_sync(cudaStream_t st, const char* what, int64_t k) {
  static const bool on = [] {
    const char* e = getenv("GF_LAUNCH_SYNC");
    return e && e[0] == '1';
  }();
  if (!on) return;
  fprintf(stderr, "[gf] k=%lld %s launched\n", (long long)k, what);
  GF_CUDA(cudaStreamSynchronize(st));
  fprintf(stderr, "[gf] k=%lld %s done\n", (long long)k, what);
}

template <typename T>
static void launch_step(gf_solver* s, int64_t k, cudaStream_t st) {
  gf_matrix* A = s->S->A;
  gf_projector* P = s->S->P;
  Ctl* ctl = s->ctl.as<Ctl>();
  if (k > 0 && s->indirect) {
    // Indirect projection of iteration k-1 (solver.py:397-411): CGLS on
    // (I + A'A) x = c_x + A' c_y warm-started at x^, tolerance from the
    // decreasing schedule min(1e-2, max(1e-10, 0.1 * drift)) unless fixed.
    Ctl h;
    GF_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    double drift = 0.0;
    GF_CUDA(cudaMemcpyAsync(&drift, s->hist.as<double>() + (k - 1) * 8 + 6, sizeof(double), cudaMemcpyDeviceToHost,
                            st));
    GF_CUDA(cudaStreamSynchronize(st));
    if (h.status != GF_STATUS_RUNNING) return;
    const double ptol = s->ptol > 0.0 ? s->ptol : std::min(1e-2, std::max(1e-10, 0.1 * drift));
    GF_CUDA(cudaMemcpyAsync(s->xplus.p, s->xk.p, s->n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    bool ok = false;
    const int64_t inner = cgls_solve(s->S->A, true, s->S->comm, s->cy.as<double>(), s->cx.as<double>(),
                                     s->xplus.as<double>(), ptol, P->max_inner, &ok, st);
    GF_CUDA(cudaMemcpyAsync(&ctl->inner, &inner, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    x_wide_kernel<T><<<(unsigned)s->grid_s, 256, 0, st>>>(make_xepi<T>(s), s->xplus.as<double>(),
                                                            s->xpart.as<double>(), 0, nullptr, nullptr);
    GF_CHECK_LAUNCH();
    GF_CUDA(cudaStreamSynchronize(st));   // `inner` lives on this stack frame
    s->launches += 1;
  } else if (k > 0) {  // S(k-1): x+ = Ginv rhs and the x side of iteration k
    s->mark(0, st, true);
    if (s->splan.ok) sym_go<T>(s, st, false);
    else if (s->rplan.ok) ring_dispatch<T>(s, st, false);
    else
    launch_k(use_pdl(s), rowgemv_kernel<T, 1, XEpi<T>>, dim3((unsigned)s->grid_s), dim3(kRowThreads), 0, st,
             (const T*)P->ginv.as<T>(), s->q, s->ldq, (const T*)s->rhs_T.as<T>(), (const T*)s->rhs_T.as<T>(),
             make_xepi<T>(s), s->xpart.as<double>());
    GF_CHECK_LAUNCH();
    s->mark(0, st, false);
    s->launches += 1;
    dbg_sync(st, "S", k);
  }
  if (s->m > 0 && (s->fplan.ok || s->fplan2.ok)) {
    // one pass over A_hat (row pass + y side + column pass) carrying the Z
    // step: alone on one GPU; under a communicator the column sums and y
    // scalars, then the all-reduce and the rest of the Z step
    s->mark(7, st, true);
    if (s->fplan.ok) launch_fused<T>(s, st);
    else fused2_dispatch<T>(s, st, false);   // rows split over the CTAs of a cluster
    s->mark(7, st, false);
    s->launches += 1;
    dbg_sync(st, "fused", k);
    if (!comm_active(s->S->comm)) return;
    s->mark(6, st, true);
    allreduce_sum(s->S->comm, s->red.as<double>(), 2 * s->ld + kScal, st);
    s->mark(6, st, false);
    s->mark(5, st, true);
    const unsigned g = (unsigned)(s->fplan.ok ? s->fplan.grid : s->fplan2.grid);
    const int64_t slabs = s->fplan.ok ? s->fplan.grid : s->fplan2.grid / s->fplan2.cl;
    const int64_t nrpart = s->fplan.ok ? (int64_t)s->fplan.ne * s->fplan.grid : (int64_t)s->fplan2.ne * s->fplan2.grid;
    zfinish_kernel<T><<<g, kTailThreads, 0, st>>>(make_ztail<T>(s, slabs, nrpart));
    GF_CHECK_LAUNCH();
    s->mark(5, st, false);
    s->launches += 1;
    return;
  }
  if (s->m > 0) {
    int64_t slabs, nrpart;
    {             // two passes: row pass (+ y side), then column pass
      s->mark(1, st, true);
      rowgemv_kernel<T, 2, YEpi<T>><<<(unsigned)s->grid_r, kRowThreads, 0, st>>>(
          (const T*)A->data, s->m, s->ld, s->xk_T.as<T>(), s->xh_T.as<T>(), make_yepi<T>(s), s->rpart.as<double>());
      GF_CHECK_LAUNCH();
      s->mark(1, st, false);
      s->mark(2, st, true);
      colgemv_kernel<T, 2, false><<<dim3((unsigned)s->cplan.col_blocks, (unsigned)s->cplan.slabs), kColThreads, 0, st>>>(
          (const T*)A->data, s->m, s->ld, s->cy.as<double>(), s->nuh2.as<double>() + (k & 1) * s->m,
          s->cplan.rows_per_slab, s->cpart.as<double>(), &ctl->status);
      GF_CHECK_LAUNCH();
      s->mark(2, st, false);
      slabs = s->cplan.slabs;
      nrpart = s->grid_r;
      s->launches += 2;
    }
    if (!comm_active(s->S->comm)) {   // Z(k) in one launch: slab + y reduce + controller
      s->mark(5, st, true);
      launch_k(use_pdl(s), zslab_tall_kernel<T, true>, dim3((unsigned)s->grid_zt), dim3(256), 0, st, ctl, s->prm,
               (const double*)s->cpart.as<double>(), slabs, s->ld, s->n, (const double*)s->rpart.as<double>(),
               nrpart, (const double*)s->cx.as<double>(), (const double*)s->S->e.as<double>(),
               (const double*)s->muh2.as<double>(), s->rhs_T.as<T>(), s->zpart.as<double>(),
               (const double*)s->xpart.as<double>(), s->grid_s, s->hist.as<double>(), s->red.as<double>());
      GF_CHECK_LAUNCH();
      s->mark(5, st, false);
      s->launches += 1;
      return;
    }
    s->mark(3, st, true);
    zreduce_kernel<<<(unsigned)s->grid_zt, 256, 0, st>>>(ctl, s->cpart.as<double>(), slabs, s->ld, s->n,
                                                          s->rpart.as<double>(), nrpart, s->red.as<double>());
    GF_CHECK_LAUNCH();
    s->mark(3, st, false);
    s->launches += 1;
  } else {
    GF_CUDA(cudaMemsetAsync(s->red.p, 0, (2 * s->ld + kScal) * sizeof(double), st));
  }
  if (comm_active(s->S->comm)) {
    s->mark(6, st, true);
    allreduce_sum(s->S->comm, s->red.as<double>(), 2 * s->ld + kScal, st);
    s->mark(6, st, false);
  }
  s->mark(5, st, true);
  zslab_tall_kernel<T, false><<<(unsigned)s->grid_zt, 256, 0, st>>>(
      ctl, s->prm, nullptr, 0, s->ld, s->n, nullptr, 0, s->cx.as<double>(), s->S->e.as<double>(),
      s->muh2.as<double>(), s->rhs_T.as<T>(), s->zpart.as<double>(), s->xpart.as<double>(), s->grid_s,
      s->hist.as<double>(), s->red.as<double>());
  GF_CHECK_LAUNCH();
  s->mark(5, st, false);
  s->launches += 1;
}

// Wide step k (m < n): R(k) row pass [A c_x, A x^_1/2] + y side + rhs;
// S(k) w = Ginv rhs, y+ = c_y + w; C(k) A' [w, nu^]; slab reduce; Z(k)
// controller; X(k) x+ = c_x - A' w and the x side of iteration k+1.
template <typename T>
static void launch_step_wide(gf_solver* s, int64_t k, cudaStream_t st) {
  gf_matrix* A = s->S->A;
  gf_projector* P = s->S->P;
  Ctl* ctl = s->ctl.as<Ctl>();
  YEpiW<T> ye;
  ye.ctl = ctl; ye.f = s->f.view; ye.d = s->S->d.as<double>();
  ye.yk = s->yk.as<double>(); ye.yt = s->yt.as<double>(); ye.cy = s->cy.as<double>();
  ye.yh2 = s->yh2.as<double>(); ye.nuh2 = s->nuh2.as<double>(); ye.ypl = s->ypl.as<double>();
  ye.rhs_T = s->rhs_T.as<T>(); ye.m = s->m; ye.alpha = s->prm.alpha; ye.gap = s->prm.gap;
  s->mark(1, st, true);
  rowgemv_kernel<T, 2, YEpiW<T>><<<(unsigned)s->grid_r, kRowThreads, 0, st>>>(
      (const T*)A->data, s->m, s->ld, s->xk_T.as<T>(), s->xh_T.as<T>(), ye, s->rpart.as<double>());
  GF_CHECK_LAUNCH();
  s->mark(1, st, false);
  if (s->indirect) {
    // Indirect projection of iteration k (projection.py:152-161, solver.py:
    // 397-411): CGLS on (I + A A') w = A c_x - c_y warm-started at
    // z0 = y^ - c_y, tolerance from the drift schedule unless fixed; then
    // y+ = c_y + w, and x+ = c_x - A' w comes from the column pass.  Like the
    // direct wide step it runs before the controller (a solve that stops at
    // k discards it).  The reference's tolerance schedule stalls wide
    // problems at MaxIterations: reproduced, not fixed.
    double hs[2] = {0.0, 0.0};
    wide_drift_kernel<<<1, 256, 0, st>>>(ctl, s->rpart.as<double>(), s->grid_r, s->xpart.as<double>(), s->grid_s,
                                         s->xplus.as<double>());
    GF_CHECK_LAUNCH();
    GF_CUDA(cudaMemcpyAsync(hs, s->xplus.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    GF_CUDA(cudaStreamSynchronize(st));
    if ((int)hs[1] == GF_STATUS_RUNNING) {
      const double ptol = s->ptol > 0.0 ? s->ptol : std::min(1e-2, std::max(1e-10, 0.1 * hs[0]));
      DBuf negcy(std::max<int64_t>(s->m, 1) * sizeof(double));
      neg_diff_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(s->m, 256), 1024)), 256, 0, st>>>(
          s->yk.as<double>(), s->cy.as<double>(), s->wv.as<double>(), negcy.as<double>(), s->m);
      GF_CHECK_LAUNCH();
      bool ok = false;
      const int64_t inner = cgls_solve(A, false, s->S->comm, s->cx.as<double>(), negcy.as<double>(),
                                       s->wv.as<double>(), ptol, P->max_inner, &ok, st);
      s->inner_host = inner;
      GF_CUDA(cudaMemcpyAsync(&ctl->inner, &s->inner_host, sizeof(int64_t), cudaMemcpyHostToDevice, st));
      wide_cgls_finish_kernel<<<(unsigned)s->grid_s, 256, 0, st>>>(s->cy.as<double>(), s->wv.as<double>(),
                                                                  s->ypl.as<double>(), s->m, s->spart.as<double>());
      GF_CHECK_LAUNCH();
      GF_CUDA(cudaStreamSynchronize(st));   // negcy and the H2D source
    }
  } else {
    WEpi we{ctl, s->cy.as<double>(), s->wv.as<double>(), s->ypl.as<double>()};
    s->mark(0, st, true);
    rowgemv_kernel<T, 1, WEpi><<<(unsigned)s->grid_s, kRowThreads, 0, st>>>(
        P->ginv.as<T>(), s->q, s->ldq, s->rhs_T.as<T>(), s->rhs_T.as<T>(), we, s->spart.as<double>());
    GF_CHECK_LAUNCH();
    s->mark(0, st, false);
  }
  s->mark(2, st, true);
  colgemv_kernel<T, 2, false><<<dim3((unsigned)s->cplan.col_blocks, (unsigned)s->cplan.slabs), kColThreads, 0, st>>>(
      (const T*)A->data, s->m, s->ld, s->wv.as<double>(), s->nuh2.as<double>() + (k & 1) * s->m,
      s->cplan.rows_per_slab, s->cpart.as<double>(), &ctl->status);
  GF_CHECK_LAUNCH();
  s->mark(2, st, false);
  s->mark(3, st, true);
  colreduce_kernel<<<dim3((unsigned)ceil_div(s->ld, 32), 2), dim3(32, 8), 0, st>>>(
      s->cpart.as<double>(), s->cplan.slabs, s->ld, 2, s->red.as<double>(), &ctl->status);
  GF_CHECK_LAUNCH();
  s->mark(3, st, false);
  s->mark(4, st, true);
  y_scalars_kernel<<<1, 256, 0, st>>>(s->rpart.as<double>(), s->grid_r, s->red.as<double>() + 2 * s->ld, ctl);
  GF_CHECK_LAUNCH();
  s->mark(4, st, false);
  s->mark(5, st, true);
  control_wide_kernel<<<(unsigned)s->grid_z, 256, 0, st>>>(
      ctl, s->prm, s->red.as<double>(), s->ld, s->n, s->cx.as<double>(), s->S->e.as<double>(), s->muh2.as<double>(),
      s->zpart.as<double>(), s->xpart.as<double>(), s->grid_s, s->hist.as<double>(), s->spart.as<double>(),
      s->grid_s);
  GF_CHECK_LAUNCH();
  s->mark(5, st, false);
  s->mark(0, st, true);
  x_wide_kernel<T><<<(unsigned)s->grid_s, 256, 0, st>>>(make_xepi<T>(s), s->red.as<double>(), s->xpart.as<double>(),
                                                          1, s->xkp.as<double>(), s->xtp.as<double>());
  GF_CHECK_LAUNCH();
  s->mark(0, st, false);
  s->launches += 7;
}

template <typename T>
static void solver_init(gf_solver* s, const double* x0, const double* nu0, double rho0, cudaStream_t st) {
  const int64_t n = s->n, m = s->m;
  DBuf x0d, nu0d, nuhat0;
  if (x0) { x0d.alloc(n * sizeof(double)); copy_in(x0d.as<double>(), x0, n, st); }
  if (nu0) { nu0d.alloc(std::max<int64_t>(m, 1) * sizeof(double)); copy_in(nu0d.as<double>(), nu0, m, st); }
  nuhat0.alloc(std::max<int64_t>(m, 1) * sizeof(double));
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(std::max(n, m), 256), 2048));
  warm_init_kernel<<<g, 256, 0, st>>>(x0 ? x0d.as<double>() : nullptr, nu0 ? nu0d.as<double>() : nullptr,
                                      s->S->e.as<double>(), s->S->d.as<double>(), n, m, rho0, s->xk.as<double>(),
                                      nuhat0.as<double>(), s->yt.as<double>());
  GF_CHECK_LAUNCH();
  GF_CUDA(cudaMemsetAsync(s->xt.p, 0, n * sizeof(double), st));
  GF_CUDA(cudaMemsetAsync(s->yk.p, 0, std::max<int64_t>(m, 1) * sizeof(double), st));
  if (nu0) {  // x~ = A_hat' nu^0 / rho (all-reduced under a row partition)
    DBuf tmp(s->ld * sizeof(double));
    GF_CUDA(cudaMemsetAsync(tmp.p, 0, s->ld * sizeof(double), st));
    if (m > 0) matvec(s->S->A, true, nuhat0.as<double>(), tmp.as<double>(), st);
    if (comm_active(s->S->comm)) allreduce_sum(s->S->comm, tmp.as<double>(), n, st);
    div_into<<<g, 256, 0, st>>>(tmp.as<double>(), n, rho0, s->xt.as<double>());
    GF_CHECK_LAUNCH();
  }
  // wide warm start: y^ = A_hat x^0 (solver.py:302); the tall row pass of
  // iteration 0 computes it on the fly instead (YEpi warm_x)
  if (x0 && !s->tall && m > 0) matvec(s->S->A, false, s->xk.as<double>(), s->yk.as<double>(), st);
  x_init_kernel<T><<<(unsigned)s->grid_s, 256, 0, st>>>(make_xepi<T>(s), s->xpart.as<double>());
  GF_CHECK_LAUNCH();
  GF_CUDA(cudaStreamSynchronize(st));
}

static void read_ctl(gf_solver* s, cudaStream_t st) {
  GF_CUDA(cudaMemcpyAsync(s->pinned, s->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  s->host = *s->pinned;
}

static void fill_state(gf_solver* s, gf_solver_state* st) {
  const Ctl& c = s->host;
  st->status = c.status;
  st->iterations = c.status == GF_STATUS_RUNNING ? c.last_good + 1 : c.iterations;
  st->k = c.last_good;
  const bool rec = c.last_good >= 0;
  st->r_pri = rec ? c.r_pri : INFINITY;
  st->r_dual = rec ? c.r_dual : INFINITY;
  st->eps_pri = rec ? c.eps_pri : NAN;
  st->eps_dual = rec ? c.eps_dual : NAN;
  st->objective = c.objective;
  st->rho = c.rho;
  st->final_rho = c.status == GF_STATUS_RUNNING ? c.rho : c.final_rho;
  st->inner_iterations = c.inner;
  st->gap = c.gap_set ? c.gap : NAN;
  st->gap_valid = c.gap_set ? 1 : 0;
}

}  // namespace gf

// ---------------------------------------------------------- C++ entry points
gf_solver* solver_create(gf_setup* S, const gf_terms* f, const gf_terms* g, const gf_settings* st_in,
                         const double* x0, const double* nu0, cudaStream_t st) {
  GF_REQUIRE(S->P != nullptr, GF_E_PARAMETER, "setup has no projector");
  GF_REQUIRE(S->P->tall || !comm_active(S->comm), GF_E_UNSUPPORTED,
             "wide (m < n) problems are solved on one GPU (row partitions need m >= n)");
  std::unique_ptr<gf_solver> s(new gf_solver());
  s->S = S;
  s->tall = S->P->tall;
  s->indirect = S->P->mode == 1;
  s->ptol = st_in->projection_tol;
  gf_matrix* A = S->A;
  s->dtype = A->dtype;
  s->m = A->m; s->n = A->n; s->ld = A->ld; s->q = S->P->q; s->ldq = S->P->ldq;
  GF_REQUIRE(f->n == s->m, GF_E_DIMENSION, "f length does not match the rows of A");
  GF_REQUIRE(g->n == s->n, GF_E_DIMENSION, "g length does not match the columns of A");
  s->prm = Params{st_in->abs_tol, st_in->rel_tol, st_in->alpha, st_in->delta, st_in->tau, st_in->max_iter,
                  st_in->adaptive_rho, 0};
  s->f.load(f, st);
  s->g.load(g, st);
  // gap stopping needs closed-form conjugates of every term; otherwise the
  // reference's gap is None and never stops (problem.py:79-84)
  if (st_in->gap_stop) {
    bool ok = conj_supported(s->f.view, s->m, st) && conj_supported(s->g.view, s->n, st);
    if (comm_active(S->comm)) {
      // f is row-partitioned: every rank must take the same decision, or
      // ranks that test a partial gap stop while the others wait in the next
      // all-reduce
      DBuf flag(sizeof(double));
      const double bad = ok ? 0.0 : 1.0;
      GF_CUDA(cudaMemcpyAsync(flag.p, &bad, sizeof(double), cudaMemcpyHostToDevice, st));
      allreduce_sum(S->comm, flag.as<double>(), 1, st);
      double tot = 0.0;
      GF_CUDA(cudaMemcpyAsync(&tot, flag.p, sizeof(double), cudaMemcpyDeviceToHost, st));
      GF_CUDA(cudaStreamSynchronize(st));
      ok = tot == 0.0;
    }
    s->prm.gap = ok ? 1 : 0;
  }
  const int sms = num_sms();
  const int64_t n = s->n, m1 = std::max<int64_t>(s->m, 1), es = A->esize();
  s->grid_r = row_grid(m1, sms);
  s->grid_s = s->dtype == GF_F32 ? ginv_grid<float>(s->q, sms) : ginv_grid<double>(s->q, sms);
  s->grid_z = std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 2 * (int64_t)sms));
  s->grid_zt = std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 32), 4 * (int64_t)sms));
  s->cplan = plan_cols(m1, s->ld, s->dtype == GF_F32 ? 4 : 2, sms);
  auto vec = [&](DBuf& b, int64_t len) { b.alloc(len * sizeof(double)); GF_CUDA(cudaMemsetAsync(b.p, 0, b.bytes, st)); };
  vec(s->xk, n); vec(s->xt, n); vec(s->cx, n); vec(s->xh2, 2 * n); vec(s->muh2, 2 * n);
  vec(s->yk, m1); vec(s->yt, m1); vec(s->cy, m1); vec(s->yh2, 2 * m1); vec(s->nuh2, 2 * m1);
  auto tv = [&](DBuf& b, int64_t len) { b.alloc(len * es); GF_CUDA(cudaMemsetAsync(b.p, 0, b.bytes, st)); };
  tv(s->xk_T, s->ld); tv(s->xh_T, s->ld); tv(s->rhs_T, std::max(s->ld, s->ldq));
  {
    int dev = 0, optin = 0;
    GF_CUDA(cudaGetDevice(&dev));
    GF_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    {   // (the indirect projector has no G^-1: ldq is 0)
      const char* renv = getenv("GF_DISABLE_RING");
      if (!(renv && renv[0] == '1') && s->tall && !s->indirect && s->ldq > 0)
        s->rplan = plan_ring(s->q, s->ldq, (int)es, sms, (size_t)optin, s->grid_s);
    }
    if (s->rplan.ok) {
      if (s->dtype == GF_F32) ring_dispatch<float>(s.get(), nullptr, true);
      else ring_dispatch<double>(s.get(), nullptr, true);
    }
    {   // the lower-triangle S step (gf_sym.cuh) replaces both when it fits
      // Default: where the triangle's saved bytes pay -- G^-1 of 256 MB and
      // more (C3's q = 20000 fp64: 0.52 -> 0.29 ms; C2's q = 10000 fp32:
      // 67 -> 61 us); at q = 5000 (100 MB) the ring is as fast (24.7 vs
      // 25.9 us) and has no grid barrier.
      // GF_SYM=1 forces it on, GF_DISABLE_SYM=1 off.
      const char* senv = getenv("GF_DISABLE_SYM");
      const char* fenv = getenv("GF_SYM");
      bool want_sym = (double)s->q * (double)s->ldq * (double)es >= (double)(256ull << 20);
      if (fenv && fenv[0] == '1') want_sym = true;
      if (senv && senv[0] == '1') want_sym = false;
      if (want_sym && s->tall && !s->indirect && s->ldq > 0)
        s->splan = plan_sym(s->q, s->ldq, (int)es, sms, (size_t)optin, s->grid_s);
      if (s->splan.ok) {
        s->sym_tm = sym_map(s->S->P->ginv.p, s->q, s->ldq, s->dtype);
        s->sympart.alloc((size_t)s->splan.nt * 2 * kSymTB * sizeof(double));
        if (s->dtype == GF_F32) sym_go<float>(s.get(), nullptr, true);
        else sym_go<double>(s.get(), nullptr, true);
      }
    }
    // GF_FUSED_MAXSLOTS (dev): cap the ring slots -- compute-sanitizer's
    // synccheck tracks a bounded number of mbarriers per CTA
    // (tools/san/mbar_sanity.cu), so its runs use small rings
    const char* ms_env = getenv("GF_FUSED_MAXSLOTS");
    const int max_slots = ms_env ? std::max(4, atoi(ms_env)) : kMaxSlots;
    s->fplan = plan_fused(s->m, s->ld, (int)es, sms, (size_t)optin, max_slots);
    const char* env = getenv("GF_DISABLE_FUSED");
    if ((env && env[0] == '1') || !s->tall) s->fplan.ok = false;
    // With only one row per group (rows of ~40 KB and more: five ring slots)
    // the fused pass is bound by the per-row fp64 epilogue latency rather
    // than by HBM, and the two-pass schedule -- whose row pass runs the
    // epilogues 32 rows per warp across thousands of warps -- is faster:
    // measured C2 logistic 100000 x 10000 fp32 1.52 vs 1.85 ms, SVM
    // 200000 x 5000 fp64 2.54 vs 2.85 ms per iteration.
    const char* force = getenv("GF_FORCE_FUSED");   // dev override for measurements
    const bool one_row = s->fplan.tr == 1 || !s->fplan.ok;
    if (s->fplan.ok && s->fplan.tr == 1 && !(force && force[0] == '1')) s->fplan.ok = false;
    if (s->fplan.ok) {
      if (s->dtype == GF_F32) fused_prepare<float>(s.get());
      else fused_prepare<double>(s.get());
    }
    // Rows of 40 KB and more: split each row over the CTAs of a cluster
    // (gf_fused.cuh, fused_rowcol_cl_kernel) -- of the cluster sizes (2, 4,
    // 8 or 9 CTAs) that leave two rows per group and <= 5 vectors per thread,
    // the one with the most co-resident SMs: 2 for fp64 n = 5000 / fp32
    // n = 10000, 4 for fp64 n = 10000, 9 for fp64 n = 20000 (C3; 8 would
    // leave 28 SMs idle).  GF_FUSED_CL2=0 disables it, =1 forces it for any
    // tall shape (measurements); GF_FUSED_CL=c picks the cluster size.
    // Newton-prox losses (logistic, negative entropy: ~8 fp64 Newton steps
    // per row, up to 100) take the lagged variant (kNewtonLag): with the rows
    // kept in shared memory every slow prox stalls its cluster's stream
    // (C2 logistic 100000 x 10000 fp32: 1.35 ms, vs 1.32 ms two-pass); with
    // the column pass re-reading rows from L2 kNewtonLag groups behind and
    // seven epilogue warps, 0.95 ms.  GF_FUSED_LAG=0 turns it off (two-pass),
    // =1 forces it for any loss (tests).  2-CTA clusters only: fp64 n = 10000
    // stays two-pass.
    const char* cl2env = getenv("GF_FUSED_CL2");
    const char* clenv = getenv("GF_FUSED_CL");
    const bool cl2_off = cl2env && cl2env[0] == '0', cl2_force = cl2env && cl2env[0] == '1';
    const char* lagenv = getenv("GF_FUSED_LAG");
    const bool newton = s->tall && !cl2_force && !cl2_off && one_row && !s->fplan.ok &&
                        has_newton_prox(s->f.view, s->m, st);
    const bool lag_on = lagenv ? lagenv[0] == '1' : newton;
    if (s->tall && !cl2_off && (!newton || lag_on) && (cl2_force || (one_row && !s->fplan.ok)) &&
        !(env && env[0] == '1')) {
      const int lag = lag_on ? kNewtonLag : 0;
      // every cluster size that fits; the one that keeps the most SMs busy
      // wins (a larger cluster only for >= 5 % more: its exchange costs more).
      // Co-resident clusters of c CTAs on a 148-SM B200 (one CTA per SM,
      // tools/cluster_probe.cu): 2 -> 148 SMs, 4 -> 132, 8 -> 120, 9 -> 135.
      FusedPlan2 best;
      for (int cl : {2, 4, 8, 9}) {
        if ((clenv && atoi(clenv) != cl) || (lag && cl != 2)) continue;
        s->fplan2 = plan_fused_cl(s->m, s->ld, (int)es, sms, (size_t)optin, sms / cl, cl, max_slots, lag);
        if (!s->fplan2.ok || (s->fplan2.tr < 2 && !cl2_force)) continue;
        const int ncl = s->dtype == GF_F32 ? fused2_dispatch<float>(s.get(), nullptr, true)
                                           : fused2_dispatch<double>(s.get(), nullptr, true);
        s->fplan2 = plan_fused_cl(s->m, s->ld, (int)es, sms, (size_t)optin, ncl, cl, max_slots, lag);
        if (s->fplan2.ok && (!best.ok || 20 * (int64_t)s->fplan2.grid >= 21 * (int64_t)best.grid)) best = s->fplan2;
      }
      s->fplan2 = best;
      if (s->fplan2.ok && (s->fplan2.tr >= 2 || cl2_force)) s->fplan.ok = false;
      else s->fplan2.ok = false;
    }
    const char* vb = getenv("GF_VERBOSE_SETUP");
    if (vb && vb[0] == '1') {
      if (s->fplan.ok)
        fprintf(stderr, "[gf] iteration: fused pass, grid %d, %d compute warps, %d rows per group, %d slots\n",
                s->fplan.grid, s->fplan.cw, s->fplan.tr, s->fplan.nslot);
      else if (s->fplan2.ok)
        fprintf(stderr, "[gf] iteration: cluster pass, %d-CTA clusters, grid %d, %d rows per group, %d slots, lag %d\n",
                s->fplan2.cl, s->fplan2.grid, s->fplan2.tr, s->fplan2.nslot, s->fplan2.lag);
      else
        fprintf(stderr, "[gf] iteration: two-pass schedule\n");
    }
  }
  const int64_t nslab = std::max<int64_t>({s->cplan.slabs, s->fplan.ok ? s->fplan.grid : 1,
                                           s->fplan2.ok ? s->fplan2.grid / s->fplan2.cl : 1});
  vec(s->rpart, std::max<int64_t>({s->grid_r, s->fplan.ok ? kFusedEpiMax * s->fplan.grid : 1,
                                   s->fplan2.ok ? kFusedEpiMax * s->fplan2.grid : 1}) * (kRedY + 1));
  vec(s->xpart, s->grid_s * (kRedX + 1));
  vec(s->zpart, std::max<int64_t>({s->grid_z, s->grid_zt, s->fplan.ok ? s->fplan.grid : 1,
                                   s->fplan2.ok ? s->fplan2.grid : 1}));
  vec(s->red, 2 * s->ld + 2 * kScal + kRedX + 1);   // + CTA 0's record sums (Z step)
  if (!s->tall) {
    vec(s->ypl, m1);
    vec(s->wv, m1);
    vec(s->spart, s->grid_s);
    vec(s->xkp, n);
    vec(s->xtp, n);
  }
  if (s->indirect) vec(s->xplus, std::max<int64_t>(n, 2));
  s->cpart.alloc((size_t)nslab * 2 * s->ld * sizeof(double));
  const int64_t hrows = std::max<int64_t>(s->prm.max_iter, 1) + 1;
  vec(s->hist, hrows * 8);
  s->ctl.alloc(sizeof(Ctl));
  Ctl c{};
  c.status = GF_STATUS_RUNNING;
  c.k = 0; c.iterations = 0; c.last_good = -1;
  c.rho = st_in->rho0; c.rho_prev = st_in->rho0; c.ratio = 1.0; c.final_rho = st_in->rho0;
  c.r_pri = INFINITY; c.r_dual = INFINITY;
  GF_CUDA(cudaMemcpyAsync(s->ctl.p, &c, sizeof(Ctl), cudaMemcpyHostToDevice, st));
  s->pinned = pinned_acquire();
  GF_CUDA(cudaEventCreateWithFlags(&s->ev_done[0], cudaEventDisableTiming));
  GF_CUDA(cudaEventCreateWithFlags(&s->ev_done[1], cudaEventDisableTiming));
  GF_CUDA(cudaEventCreate(&s->ev_a));
  GF_CUDA(cudaEventCreate(&s->ev_b));
  s->warm_x = x0 != nullptr;
  if (s->dtype == GF_F32) solver_init<float>(s.get(), x0, nu0, st_in->rho0, st);
  else solver_init<double>(s.get(), x0, nu0, st_in->rho0, st);
  // objective of the all-zero half iterate (reported when iteration 0 is degenerate)
  {
    DBuf z(std::max(n, m1) * sizeof(double));
    GF_CUDA(cudaMemsetAsync(z.p, 0, z.bytes, st));
    const double obj0 = evaluate(s->f.view, s->m, z.as<double>(), st) + evaluate(s->g.view, n, z.as<double>(), st);
    GF_CUDA(cudaMemcpyAsync(&s->ctl.as<Ctl>()->objective, &obj0, sizeof(double), cudaMemcpyHostToDevice, st));
  }
  read_ctl(s.get(), st);
  return s.release();
}

void solver_run(gf_solver* s, int64_t steps, gf_solver_state* out, cudaStream_t st) {
  const int64_t last_step = s->prm.max_iter;  // step max_iter is the final projection check
  int64_t budget = steps > 0 ? steps : INT64_MAX;
  int64_t chunk = 1;
  read_ctl(s, st);
  // Two chunks in flight: chunk c+1 is enqueued before the host waits for the
  // controller snapshot of chunk c, so the GPU never idles on the round trip.
  // Kernels of steps after termination return at entry (status check).
  Ctl* snap[2] = {s->pinned, s->pinned + 1};
  cudaEvent_t done[2] = {s->ev_done[0], s->ev_done[1]};
  int inflight = 0, cur = 0;
  bool stop = s->host.status != GF_STATUS_RUNNING;
  GF_CUDA(cudaEventRecord(s->ev_a, st));
  while (!stop && s->next_step <= last_step && budget > 0) {
    const int64_t nlaunch = std::min({chunk, budget, last_step - s->next_step + 1});
    for (int64_t i = 0; i < nlaunch; ++i) {
      if (s->tall) {
        if (s->dtype == GF_F32) launch_step<float>(s, s->next_step, st);
        else launch_step<double>(s, s->next_step, st);
      } else if (s->next_step < s->prm.max_iter) {   // the wide controller ends at max_iter - 1
        if (s->dtype == GF_F32) launch_step_wide<float>(s, s->next_step, st);
        else launch_step_wide<double>(s, s->next_step, st);
      }
      ++s->next_step;
    }
    GF_CUDA(cudaMemcpyAsync(snap[cur], s->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    GF_CUDA(cudaEventRecord(done[cur], st));
    budget -= nlaunch;
    ++inflight;
    chunk = std::min<int64_t>(chunk * 2, 32);
    if (inflight == 2 || budget <= 0 || s->next_step > last_step) {
      const int prev = cur ^ (inflight == 2 ? 1 : 0);   // oldest chunk in flight
      GF_CUDA(cudaEventSynchronize(done[prev]));
      --inflight;
      s->host = *snap[prev];
      stop = s->host.status != GF_STATUS_RUNNING;
    }
    cur ^= 1;
  }
  GF_CUDA(cudaEventRecord(s->ev_b, st));
  GF_CUDA(cudaStreamSynchronize(st));
  read_ctl(s, st);
  s->collect();
  float ms = 0.f;
  GF_CUDA(cudaEventElapsedTime(&ms, s->ev_a, s->ev_b));
  s->elapsed_ms += ms;
  fill_state(s, out);
}

void solver_history(gf_solver* s, int64_t count, double* out, cudaStream_t st) {
  std::vector<double> h(std::max<int64_t>(count, 1) * 8);
  if (count > 0) {
    GF_CUDA(cudaMemcpyAsync(h.data(), s->hist.p, count * 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
    GF_CUDA(cudaStreamSynchronize(st));
  }
  for (int64_t k = 0; k < count; ++k)
    for (int c = 0; c < 6; ++c) out[k * 6 + c] = h[k * 8 + c];
}

void solver_snapshot(gf_solver* s, double* x_hat, double* y_hat, double* xt, double* yt, double* xhh, double* yhh,
                     cudaStream_t st) {
  DBuf bx(std::max<int64_t>(s->n, 1) * sizeof(double)), by(std::max<int64_t>(s->m, 1) * sizeof(double));
  snapshot_kernel<<<64, 256, 0, st>>>(s->ctl.as<Ctl>(), s->n, s->m, s->xh2.as<double>(), s->yh2.as<double>(),
                                      s->S->e.as<double>(), s->S->d.as<double>(), bx.as<double>(), by.as<double>());
  GF_CHECK_LAUNCH();
  // wide: a step that did not end the solve ran X(k), which already holds
  // x^ and x~ of iteration k + 1; iteration k's are in xkp / xtp
  read_ctl(s, st);
  const bool advanced = !s->tall && s->host.status == GF_STATUS_RUNNING && s->next_step > 0;
  copy_out(x_hat, (advanced ? s->xkp : s->xk).as<double>(), s->n, st);
  copy_out(y_hat, s->yk.as<double>(), s->m, st);
  copy_out(xt, (advanced ? s->xtp : s->xt).as<double>(), s->n, st);
  copy_out(yt, s->yt.as<double>(), s->m, st);
  copy_out(xhh, bx.as<double>(), s->n, st);
  copy_out(yhh, by.as<double>(), s->m, st);
  GF_CUDA(cudaStreamSynchronize(st));
}

void solver_result(gf_solver* s, double* x, double* y, double* mu, double* nu, gf_solver_state* out,
                   cudaStream_t st) {
  read_ctl(s, st);
  DBuf bx(std::max<int64_t>(s->n, 1) * sizeof(double)), bm(std::max<int64_t>(s->n, 1) * sizeof(double));
  DBuf by(std::max<int64_t>(s->m, 1) * sizeof(double)), bn(std::max<int64_t>(s->m, 1) * sizeof(double));
  result_kernel<<<64, 256, 0, st>>>(s->ctl.as<Ctl>(), s->n, s->m, s->xh2.as<double>(), s->muh2.as<double>(),
                                    s->yh2.as<double>(), s->nuh2.as<double>(), s->S->e.as<double>(),
                                    s->S->d.as<double>(), bx.as<double>(), bm.as<double>(), by.as<double>(),
                                    bn.as<double>());
  GF_CHECK_LAUNCH();
  if (x) copy_out(x, bx.as<double>(), s->n, st);
  if (mu) copy_out(mu, bm.as<double>(), s->n, st);
  if (y) copy_out(y, by.as<double>(), s->m, st);
  if (nu) copy_out(nu, bn.as<double>(), s->m, st);
  GF_CUDA(cudaStreamSynchronize(st));
  fill_state(s, out);
}

double solver_elapsed(gf_solver* s) { return s->elapsed_ms; }

void solver_stats(gf_solver* s, int64_t* launches, double* kernel_ms, int64_t* kernel_count) {
  if (launches) *launches = s->launches;
  for (int i = 0; i < 8; ++i) {
    if (kernel_ms) kernel_ms[i] = s->kms[i];
    if (kernel_count) kernel_count[i] = s->kcount[i];
  }
}

void solver_profile(gf_solver* s, int enable) {
  s->profile = enable != 0;
  for (int i = 0; i < 8; ++i) { s->kms[i] = 0.0; s->kcount[i] = 0; }
}

void solver_free(gf_solver* s) { delete s; }
