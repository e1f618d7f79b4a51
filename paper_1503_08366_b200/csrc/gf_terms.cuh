// Per-coordinate term arithmetic in fp64: prox, evaluation (device side).
//
// Restates the reference prox library (prox.py) and evaluator
// (functions.py:77-105, :307-327) as scalar __device__ functions so that every
// kernel that touches a coordinate (the fused ADMM epilogues, the standalone
// prox/evaluate kernels) runs the identical arithmetic.  Everything here is
// fp64 regardless of the matrix dtype: the term math is O(m+n) per iteration,
// and fp64 keeps the Newton tolerance (1e-12, prox.py:23) meaningful and the
// indicator sign tests identical to the reference.
#pragma once

#include <stdint.h>
#include <math.h>

namespace gf {

enum Kind : int {
  kAbs = 0, kSquare = 1, kHuber = 2, kNegEntr = 3, kLogistic = 4,
  kMaxPos0 = 5, kIndGe0 = 6, kIndLe0 = 7, kIndEq0 = 8, kZero = 9
};

constexpr double kNewtonTol = 1e-12;  // prox.py:23
constexpr int kNewtonMaxIt = 100;     // prox.py:24

// Term arrays (device pointers), structure of arrays.
struct TermsView {
  const int8_t* h;
  const double* a;
  const double* b;
  const double* c;
  const double* d;
  const double* e;
};

struct Term {
  int h;
  double a, b, c, d, e;
};

__device__ __forceinline__ Term load_term(const TermsView& t, int64_t i) {
  Term r;
  r.h = t.h[i];
  r.a = t.a[i];
  r.b = t.b[i];
  r.c = t.c[i];
  r.d = t.d[i];
  r.e = t.e[i];
  return r;
}

// Every arithmetic step below rounds like numpy does (one rounding per
// operation, no FMA contraction): the reference's safeguarded Newton can
// cycle for the full 100 iterations on some inputs, and then
// its result depends on the rounding of every step.  exp/log are CUDA's
// correctly-rounded-to-1-ulp versions.
__device__ __forceinline__ double A_(double x, double y) { return __dadd_rn(x, y); }
__device__ __forceinline__ double S_(double x, double y) { return __dsub_rn(x, y); }
__device__ __forceinline__ double M_(double x, double y) { return __dmul_rn(x, y); }
__device__ __forceinline__ double D_(double x, double y) { return __ddiv_rn(x, y); }

__device__ __forceinline__ double sgn(double v) { return (v > 0.0) - (v < 0.0); }

__device__ __forceinline__ double sigmoid(double x) { return D_(1.0, A_(1.0, exp(-x))); }

// Logistic prox: root of rho*(z-v) + sigmoid(z) in [v-1/rho, v], safeguarded
// Newton with bisection fallback, same iteration sequence as prox.py:27-48.
__device__ inline double prox_logistic(double rho, double v) {
  double lo = S_(v, D_(1.0, rho)), hi = v;
  double z = S_(v, D_(sigmoid(v), A_(rho, 0.25)));
  z = fmin(fmax(z, lo), hi);
  const double tol = M_(kNewtonTol, fmax(1.0, fabs(M_(rho, v))));
  for (int it = 0; it < kNewtonMaxIt; ++it) {
    const double s = sigmoid(z);
    const double g = A_(M_(rho, S_(z, v)), s);
    if (fabs(g) <= tol) break;
    if (g < 0.0) lo = z; else hi = z;
    double zn = S_(z, D_(g, A_(rho, M_(s, S_(1.0, s)))));
    if (zn <= lo || zn >= hi || !isfinite(zn)) zn = M_(0.5, A_(lo, hi));
    z = zn;
  }
  return z;
}

// NegEntr prox: root of log z + 1 + rho*(z-v) on z > 0 (prox.py:51-70).
__device__ inline double prox_negentr(double rho, double v) {
  double z = fmax(v, 1e-6);
  double lo = 0.0, hi = fmax(v, 1.0);
  const double tol = M_(kNewtonTol, fmax(1.0, M_(fabs(rho), A_(fabs(v), 1.0))));
  for (int it = 0; it < kNewtonMaxIt; ++it) {
    const double g = A_(A_(log(z), 1.0), M_(rho, S_(z, v)));
    if (fabs(g) <= tol) break;
    if (g < 0.0) lo = z; else hi = z;
    double zn = S_(z, D_(M_(g, z), A_(1.0, M_(rho, z))));
    if (zn <= lo || zn >= hi || !isfinite(zn)) zn = M_(0.5, A_(lo, hi));
    z = zn;
  }
  return z;
}

// Base prox argmin_z h(z) + rho/2 (z - v)^2 (prox.py:73-98).
__device__ __forceinline__ double prox_base(int kind, double rho, double v) {
  switch (kind) {
    case kAbs: return M_(sgn(v), fmax(S_(fabs(v), D_(1.0, rho)), 0.0));
    case kSquare: return D_(M_(rho, v), A_(1.0, rho));
    case kHuber:
      return fabs(v) <= A_(1.0, D_(1.0, rho)) ? D_(M_(rho, v), A_(1.0, rho)) : S_(v, D_(sgn(v), rho));
    case kNegEntr: return prox_negentr(rho, v);
    case kLogistic: return prox_logistic(rho, v);
    case kMaxPos0: {
      const double inv = D_(1.0, rho);
      return v <= 0.0 ? v : (v >= inv ? S_(v, inv) : 0.0);
    }
    case kIndGe0: return fmax(v, 0.0);
    case kIndLe0: return fmin(v, 0.0);
    case kIndEq0: return 0.0;
    default: return v;  // kZero
  }
}

// Full-term prox through the parametric transform (prox.py:129-138):
//   prox(v) = (prox_{h, (e+rho)/(c a^2)}(a (v rho - d)/(e+rho) - b) + b) / a
// with c == 0 terms acting as ZERO with c = 1 (functions.py:284-303).
__device__ __forceinline__ double prox_term(const Term& t, double rho, double v) {
  const bool zc = t.c == 0.0;
  const int kind = zc ? kZero : t.h;
  const double ceff = zc ? 1.0 : t.c;
  // x*1, x/1, x+0 (e = 0) and x-0 (d = 0) are exact in IEEE arithmetic, so
  // skipping them for unit parameters changes no bit of the result but
  // shortens the dependent fp64 chain (divisions dominate it).
  const double den = t.e == 0.0 ? rho : A_(t.e, rho);
  const double cas = M_(M_(ceff, t.a), t.a);
  const double rho_h = cas == 1.0 ? den : D_(den, cas);
  const double num = t.d == 0.0 ? M_(v, rho) : S_(M_(v, rho), t.d);
  const double z0 = S_(D_(t.a == 1.0 ? num : M_(t.a, num), den), t.b);
  const double z = prox_base(kind, rho_h, z0);
  const double zb = A_(z, t.b);
  return t.a == 1.0 ? zb : D_(zb, t.a);
}

// h(x) with +inf off-domain (functions.py:77-105).
__device__ __forceinline__ double eval_base(int kind, double x) {
  switch (kind) {
    case kAbs: return fabs(x);
    case kSquare: return M_(M_(0.5, x), x);
    case kHuber: return fabs(x) <= 1.0 ? M_(M_(0.5, x), x) : S_(fabs(x), 0.5);
    case kNegEntr: return x > 0.0 ? M_(x, log(x)) : (x == 0.0 ? 0.0 : INFINITY);
    case kLogistic: return x > 0.0 ? A_(x, log1p(exp(-x))) : log1p(exp(x));
    case kMaxPos0: return fmax(x, 0.0);
    case kIndGe0: return x >= 0.0 ? 0.0 : INFINITY;
    case kIndLe0: return x <= 0.0 ? 0.0 : INFINITY;
    case kIndEq0: return x == 0.0 ? 0.0 : INFINITY;
    default: return 0.0;  // kZero
  }
}

// Convex conjugate h*(w) of a base function, +inf off its domain
// (functions.py:108-144).
__device__ __forceinline__ double conj_base(int kind, double w) {
  switch (kind) {
    case kAbs: return fabs(w) <= 1.0 ? 0.0 : INFINITY;
    case kSquare: return M_(M_(0.5, w), w);
    case kHuber: return fabs(w) <= 1.0 ? M_(M_(0.5, w), w) : INFINITY;
    case kNegEntr: return exp(S_(w, 1.0));
    case kLogistic: {   // binary entropy on [0, 1]
      if (!(w >= 0.0 && w <= 1.0)) return INFINITY;
      const double lhs = w > 0.0 ? M_(w, log(w)) : 0.0;
      const double rhs = w < 1.0 ? M_(S_(1.0, w), log1p(-w)) : 0.0;
      return A_(lhs, rhs);
    }
    case kMaxPos0: return (w >= 0.0 && w <= 1.0) ? 0.0 : INFINITY;
    case kIndGe0: return w <= 0.0 ? 0.0 : INFINITY;
    case kIndLe0: return w >= 0.0 ? 0.0 : INFINITY;
    case kIndEq0: return 0.0;
    default: return w == 0.0 ? 0.0 : INFINITY;   // kZero
  }
}

// Conjugate of c*h(a x - b) + d x + (e/2) x^2 at w (functions.py:329-393).
// e == 0 reduces to h* by shift and scale; e > 0 has a closed form only for
// Zero, Square and the three indicators -- otherwise `unsupported` is set and
// the caller reports no gap (the reference returns None).
__device__ __forceinline__ double conj_term(const Term& t, double w, bool& unsupported) {
  const bool zc = t.c == 0.0;
  const int kind = zc ? kZero : t.h;
  const double c = zc ? 1.0 : t.c;
  const double a = t.a, b = t.b, e = t.e;
  const double wd = S_(w, t.d);
  if (e == 0.0) {
    const double q = D_(wd, M_(a, c));
    return A_(M_(c, conj_base(kind, q)), D_(M_(b, wd), a));
  }
  switch (kind) {
    case kZero: return D_(M_(wd, wd), M_(2.0, e));
    case kSquare: {
      const double alpha = A_(M_(M_(c, a), a), e);
      const double beta = M_(M_(-c, a), b);
      const double cst = M_(M_(M_(0.5, c), b), b);
      const double tt = S_(wd, beta);
      return S_(D_(M_(tt, tt), M_(2.0, alpha)), cst);
    }
    case kIndEq0:
    case kIndGe0:
    case kIndLe0: {
      const double x0 = D_(b, a);
      const double boundary = S_(M_(wd, x0), M_(M_(M_(0.5, e), x0), x0));
      if (kind == kIndEq0) return boundary;
      const double xbar = D_(wd, e);
      const double interior = D_(M_(wd, wd), M_(2.0, e));
      const bool feasible = kind == kIndGe0 ? (a > 0.0 ? xbar >= x0 : xbar <= x0)
                                            : (a > 0.0 ? xbar <= x0 : xbar >= x0);
      return feasible ? interior : boundary;
    }
    default:
      unsupported = true;
      return 0.0;
  }
}

// One coordinate's contribution c*h(a v - b) + d v + e v^2 / 2; zero-weight
// terms contribute no h part even off-domain (functions.py:321-324).
__device__ __forceinline__ double eval_term(const Term& t, double v) {
  const double hv = t.c == 0.0 ? 0.0 : M_(t.c, eval_base(t.h, S_(M_(t.a, v), t.b)));
  return A_(A_(hv, M_(t.d, v)), M_(M_(0.5, t.e), M_(v, v)));
}

}  // namespace gf
