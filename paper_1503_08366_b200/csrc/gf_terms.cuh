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

__device__ __forceinline__ double sgn(double v) { return (v > 0.0) - (v < 0.0); }

__device__ __forceinline__ double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

// Logistic prox: root of rho*(z-v) + sigmoid(z) in [v-1/rho, v], safeguarded
// Newton with bisection fallback, same iteration sequence as prox.py:27-48.
__device__ inline double prox_logistic(double rho, double v) {
  double lo = v - 1.0 / rho, hi = v;
  double z = v - sigmoid(v) / (rho + 0.25);
  z = fmin(fmax(z, lo), hi);
  const double tol = kNewtonTol * fmax(1.0, fabs(rho * v));
  for (int it = 0; it < kNewtonMaxIt; ++it) {
    const double s = sigmoid(z);
    const double g = rho * (z - v) + s;
    if (fabs(g) <= tol) break;
    if (g < 0.0) lo = z; else hi = z;
    double zn = z - g / (rho + s * (1.0 - s));
    if (zn <= lo || zn >= hi || !isfinite(zn)) zn = 0.5 * (lo + hi);
    z = zn;
  }
  return z;
}

// NegEntr prox: root of log z + 1 + rho*(z-v) on z > 0 (prox.py:51-70).
__device__ inline double prox_negentr(double rho, double v) {
  double z = fmax(v, 1e-6);
  double lo = 0.0, hi = fmax(v, 1.0);
  const double tol = kNewtonTol * fmax(1.0, fabs(rho) * (fabs(v) + 1.0));
  for (int it = 0; it < kNewtonMaxIt; ++it) {
    const double g = log(z) + 1.0 + rho * (z - v);
    if (fabs(g) <= tol) break;
    if (g < 0.0) lo = z; else hi = z;
    double zn = z - g * z / (1.0 + rho * z);
    if (zn <= lo || zn >= hi || !isfinite(zn)) zn = 0.5 * (lo + hi);
    z = zn;
  }
  return z;
}

// Base prox argmin_z h(z) + rho/2 (z - v)^2 (prox.py:73-98).
__device__ __forceinline__ double prox_base(int kind, double rho, double v) {
  switch (kind) {
    case kAbs: return sgn(v) * fmax(fabs(v) - 1.0 / rho, 0.0);
    case kSquare: return rho * v / (1.0 + rho);
    case kHuber:
      return fabs(v) <= 1.0 + 1.0 / rho ? rho * v / (1.0 + rho) : v - sgn(v) / rho;
    case kNegEntr: return prox_negentr(rho, v);
    case kLogistic: return prox_logistic(rho, v);
    case kMaxPos0: {
      const double inv = 1.0 / rho;
      return v <= 0.0 ? v : (v >= inv ? v - inv : 0.0);
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
  const double den = t.e + rho;
  const double rho_h = den / (ceff * t.a * t.a);
  const double z0 = t.a * (v * rho - t.d) / den - t.b;
  const double z = prox_base(kind, rho_h, z0);
  return (z + t.b) / t.a;
}

// h(x) with +inf off-domain (functions.py:77-105).
__device__ __forceinline__ double eval_base(int kind, double x) {
  switch (kind) {
    case kAbs: return fabs(x);
    case kSquare: return 0.5 * x * x;
    case kHuber: return fabs(x) <= 1.0 ? 0.5 * x * x : fabs(x) - 0.5;
    case kNegEntr: return x > 0.0 ? x * log(x) : (x == 0.0 ? 0.0 : INFINITY);
    case kLogistic: return x > 0.0 ? x + log1p(exp(-x)) : log1p(exp(x));
    case kMaxPos0: return fmax(x, 0.0);
    case kIndGe0: return x >= 0.0 ? 0.0 : INFINITY;
    case kIndLe0: return x <= 0.0 ? 0.0 : INFINITY;
    case kIndEq0: return x == 0.0 ? 0.0 : INFINITY;
    default: return 0.0;  // kZero
  }
}

// One coordinate's contribution c*h(a v - b) + d v + e v^2 / 2; zero-weight
// terms contribute no h part even off-domain (functions.py:321-324).
__device__ __forceinline__ double eval_term(const Term& t, double v) {
  const double hv = t.c == 0.0 ? 0.0 : t.c * eval_base(t.h, t.a * v - t.b);
  return hv + t.d * v + 0.5 * t.e * (v * v);
}

}  // namespace gf
