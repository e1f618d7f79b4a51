// Standalone elementwise kernels: separable prox, base prox, evaluation.
// (prox.py:101-138, functions.py:160-164, :307-327).  The same __device__
// term functions (gf_terms.cuh) run inside the fused solver epilogues.

#include "gf_internal.h"

namespace gf {

void TermsDev::load(const gf_terms* t, cudaStream_t st) {
  n = t->n;
  const size_t nd = (size_t)std::max<int64_t>(n, 1);
  const size_t h_bytes = round_up(nd, 16);
  buf.alloc(h_bytes + 5 * nd * sizeof(double));
  int8_t* h = (int8_t*)buf.p;
  double* p = (double*)((char*)buf.p + h_bytes);
  if (n > 0) {
    GF_CUDA(cudaMemcpyAsync(h, t->h, n, cudaMemcpyDefault, st));
    const double* src[5] = {t->a, t->b, t->c, t->d, t->e};
    for (int k = 0; k < 5; ++k) GF_CUDA(cudaMemcpyAsync(p + k * nd, src[k], n * sizeof(double), cudaMemcpyDefault, st));
  }
  view = TermsView{h, p, p + nd, p + 2 * nd, p + 3 * nd, p + 4 * nd};
}

__global__ void prox_kernel(TermsView t, int64_t n, const double* __restrict__ rho, const double* __restrict__ v,
                            double* __restrict__ out) {
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = prox_term(load_term(t, i), rho[i], v[i]);
}

__global__ void prox_base_kernel(int kind, int64_t n, const double* __restrict__ rho, const double* __restrict__ v,
                                 double* __restrict__ out) {
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = prox_base(kind, rho[i], v[i]);
}

__global__ void eval_base_kernel(int kind, int64_t n, const double* __restrict__ x, double* __restrict__ out) {
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = eval_base(kind, x[i]);
}

__global__ void evaluate_kernel(TermsView t, int64_t n, const double* __restrict__ v, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += eval_term(load_term(t, i), v[i]);
  s = warp_sum(s);
  __shared__ double sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < 8; ++w) tot += sh[w];
    part[blockIdx.x] = tot;
  }
}

__global__ void evaluate_final(const double* __restrict__ part, int64_t count, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int64_t i = 0; i < count; ++i) s += part[i];
    *out = s;
  }
}

__global__ void conj_base_kernel(int kind, int64_t n, const double* __restrict__ w, double* __restrict__ out) {
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = conj_base(kind, w[i]);
}

// part[block] = partial sum of conj_term; part[grid] (as bits) |= unsupported
__global__ void conjugate_kernel(TermsView t, int64_t n, const double* __restrict__ w, double* __restrict__ part,
                                 unsigned* __restrict__ unsup) {
  double s = 0.0;
  bool u = false;
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += conj_term(load_term(t, i), w[i], u);
  s = warp_sum(s);
  if (__any_sync(0xffffffffu, u) && (threadIdx.x & 31) == 0) atomicOr(unsup, 1u);
  __shared__ double sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int k = 0; k < 8; ++k) tot += sh[k];
    part[blockIdx.x] = tot;
  }
}

static unsigned egrid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 2048)); }

void prox_separable(const TermsView& t, int64_t n, const double* rho, const double* v, double* out, cudaStream_t st) {
  if (n <= 0) return;
  prox_kernel<<<egrid(n), 256, 0, st>>>(t, n, rho, v, out);
  GF_CHECK_LAUNCH();
}

void prox_base(int kind, int64_t n, const double* rho, const double* v, double* out, cudaStream_t st) {
  if (n <= 0) return;
  prox_base_kernel<<<egrid(n), 256, 0, st>>>(kind, n, rho, v, out);
  GF_CHECK_LAUNCH();
}

void eval_base(int kind, int64_t n, const double* x, double* out, cudaStream_t st) {
  if (n <= 0) return;
  eval_base_kernel<<<egrid(n), 256, 0, st>>>(kind, n, x, out);
  GF_CHECK_LAUNCH();
}

double evaluate(const TermsView& t, int64_t n, const double* v, cudaStream_t st) {
  if (n <= 0) return 0.0;
  const unsigned g = egrid(n);
  DBuf part((g + 1) * sizeof(double));
  evaluate_kernel<<<g, 256, 0, st>>>(t, n, v, part.as<double>());
  evaluate_final<<<1, 32, 0, st>>>(part.as<double>(), g, part.as<double>() + g);
  GF_CHECK_LAUNCH();
  double r = 0.0;
  GF_CUDA(cudaMemcpyAsync(&r, part.as<double>() + g, sizeof(double), cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  return r;
}

__global__ void conj_support_kernel(TermsView t, int64_t n, unsigned* __restrict__ unsup) {
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool u = false;
    (void)conj_term(load_term(t, i), 0.0, u);
    if (u) atomicOr(unsup, 1u);
  }
}

bool conj_supported(const TermsView& t, int64_t n, cudaStream_t st) {
  if (n <= 0) return true;
  DBuf flag(sizeof(unsigned));
  GF_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(unsigned), st));
  conj_support_kernel<<<egrid(n), 256, 0, st>>>(t, n, flag.as<unsigned>());
  GF_CHECK_LAUNCH();
  unsigned u = 0;
  GF_CUDA(cudaMemcpyAsync(&u, flag.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  return u == 0;
}

__global__ void newton_kind_kernel(TermsView t, int64_t n, unsigned* __restrict__ hit) {
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const Term u = load_term(t, i);
    if (u.c != 0.0 && (u.h == kLogistic || u.h == kNegEntr)) atomicOr(hit, 1u);
  }
}

bool has_newton_prox(const TermsView& t, int64_t n, cudaStream_t st) {
  if (n <= 0) return false;
  DBuf flag(sizeof(unsigned));
  GF_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(unsigned), st));
  newton_kind_kernel<<<egrid(n), 256, 0, st>>>(t, n, flag.as<unsigned>());
  GF_CHECK_LAUNCH();
  unsigned u = 0;
  GF_CUDA(cudaMemcpyAsync(&u, flag.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  return u != 0;
}

void conj_base(int kind, int64_t n, const double* w, double* out, cudaStream_t st) {
  if (n <= 0) return;
  conj_base_kernel<<<egrid(n), 256, 0, st>>>(kind, n, w, out);
  GF_CHECK_LAUNCH();
}

double conjugate(const TermsView& t, int64_t n, const double* w, bool* supported, cudaStream_t st) {
  *supported = true;
  if (n <= 0) return 0.0;
  const unsigned g = egrid(n);
  DBuf part((g + 2) * sizeof(double));
  GF_CUDA(cudaMemsetAsync(part.as<double>() + g + 1, 0, sizeof(double), st));
  conjugate_kernel<<<g, 256, 0, st>>>(t, n, w, part.as<double>(), (unsigned*)(part.as<double>() + g + 1));
  evaluate_final<<<1, 32, 0, st>>>(part.as<double>(), g, part.as<double>() + g);
  GF_CHECK_LAUNCH();
  double r[2] = {0.0, 0.0};
  GF_CUDA(cudaMemcpyAsync(r, part.as<double>() + g, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  unsigned u = 0;
  memcpy(&u, &r[1], sizeof(u));
  *supported = u == 0;
  return r[0];
}

}  // namespace gf
