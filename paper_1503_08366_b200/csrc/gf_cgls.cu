// Indirect projection: CGLS on the reduced system (reference
// projection.py:130-196).  For tall A it solves
//     min ||A z - h1||^2 + ||z - h2||^2   (h1 = d, h2 = c)  ->  x = z, y = A z
// and for wide A the mirrored problem with A' (h1 = c, h2 = -d) -> y = d + z,
// x = c - A' z.  The stopping test, breakdown test and warm starts follow the
// reference exactly; the inner loop is data-dependent, so the host drives it
// and reads three fp64 scalars per inner iteration.  Matvecs run in the
// working dtype of A (gf_gemv.cuh kernels through matvec()); vectors and dot
// products are fp64 with a deterministic reduction order.

#include "gf_internal.h"

namespace gf {

__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                           double* __restrict__ part) {
  double s = 0.0;
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  s = warp_sum(s);
  __shared__ double sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
}

__global__ void sum_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *out = s;
  }
}

// y = a*x + b*y   (elementwise, fp64)
__global__ void axpby_kernel(double a, const double* __restrict__ x, double b, double* __restrict__ y, int64_t n) {
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}

// out = x - y
__global__ void sub_kernel(const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ out,
                           int64_t n) {
  for (int64_t i = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] - y[i];
}

static unsigned vblocks(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 512)); }

struct Cgls {
  const gf_matrix* A;
  bool tall;        // orientation of A (mv = A or A')
  gf_comm* comm;    // row partition (tall only)
  cudaStream_t st;
  DBuf part, scal;
  explicit Cgls(const gf_matrix* a, bool t, gf_comm* c, cudaStream_t s) : A(a), tall(t), comm(c), st(s) {
    part.alloc(512 * sizeof(double));
    scal.alloc(8 * sizeof(double));
  }
  int64_t nz() const { return tall ? A->n : A->m; }   // unknown z
  int64_t nr() const { return tall ? A->m : A->n; }   // residual r1
  void mv(const double* z, double* out) { if (nr() > 0) matvec(A, !tall, z, out, st); }
  void rmv(const double* r, double* out) {
    if (nr() > 0) matvec(A, tall, r, out, st);
    else GF_CUDA(cudaMemsetAsync(out, 0, nz() * sizeof(double), st));
    if (tall && comm_active(comm)) allreduce_sum(comm, out, nz(), st);
  }
  // dot of two vectors; `local` marks row-sharded (r-space) vectors
  double dot(const double* a, const double* b, int64_t n, bool local) {
    const unsigned g = vblocks(n);
    double v = 0.0;
    if (n > 0) {
      dot_kernel<<<g, 256, 0, st>>>(a, b, n, part.as<double>());
      sum_kernel<<<1, 32, 0, st>>>(part.as<double>(), (int)g, scal.as<double>());
    } else {
      GF_CUDA(cudaMemsetAsync(scal.p, 0, sizeof(double), st));
    }
    GF_CHECK_LAUNCH();
    if (local && comm_active(comm)) allreduce_sum(comm, scal.as<double>(), 1, st);
    GF_CUDA(cudaMemcpyAsync(&v, scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    GF_CUDA(cudaStreamSynchronize(st));
    return v;
  }
};

// z (in: warm start, out: solution). Returns iterations; *ok = converged.
int64_t cgls_solve(const gf_matrix* A, bool tall, gf_comm* comm, const double* h1, const double* h2, double* z,
                   double tol, int64_t max_inner, bool* ok, cudaStream_t st) {
  Cgls C(A, tall, comm, st);
  const int64_t nz = C.nz(), nr = C.nr();
  DBuf r1(std::max<int64_t>(nr, 1) * 8), r2(nz * 8), s(nz * 8), p(nz * 8), q(std::max<int64_t>(nr, 1) * 8);
  const unsigned gz = vblocks(nz), gr = vblocks(nr);
  // r1 = h1 - A z ; r2 = h2 - z ; s = A' r1 + r2            (projection.py:171-173)
  C.mv(z, q.as<double>());
  if (nr > 0) sub_kernel<<<gr, 256, 0, st>>>(h1, q.as<double>(), r1.as<double>(), nr);
  sub_kernel<<<gz, 256, 0, st>>>(h2, z, r2.as<double>(), nz);
  C.rmv(r1.as<double>(), s.as<double>());
  axpby_kernel<<<gz, 256, 0, st>>>(1.0, r2.as<double>(), 1.0, s.as<double>(), nz);
  GF_CHECK_LAUNCH();
  double gamma = C.dot(s.as<double>(), s.as<double>(), nz, false);
  // ref = || A' h1 + h2 ||                                   (projection.py:175-177)
  C.rmv(h1, p.as<double>());
  axpby_kernel<<<gz, 256, 0, st>>>(1.0, h2, 1.0, p.as<double>(), nz);
  GF_CHECK_LAUNCH();
  double ref = sqrt(C.dot(p.as<double>(), p.as<double>(), nz, false));
  if (ref == 0.0) ref = 1.0;
  const double thresh = (tol * ref) * (tol * ref);
  *ok = true;
  if (gamma <= thresh) return 0;
  GF_CUDA(cudaMemcpyAsync(p.p, s.p, nz * 8, cudaMemcpyDeviceToDevice, st));
  for (int64_t it = 1; it <= max_inner; ++it) {
    C.mv(p.as<double>(), q.as<double>());                     // q = A p
    const double denom = C.dot(q.as<double>(), q.as<double>(), nr, true) +
                         C.dot(p.as<double>(), p.as<double>(), nz, false);
    if (denom <= 0.0 || !std::isfinite(denom)) { *ok = false; return it; }
    const double alpha = gamma / denom;
    axpby_kernel<<<gz, 256, 0, st>>>(alpha, p.as<double>(), 1.0, z, nz);                       // z += a p
    if (nr > 0) axpby_kernel<<<gr, 256, 0, st>>>(-alpha, q.as<double>(), 1.0, r1.as<double>(), nr);  // r1 -= a q
    axpby_kernel<<<gz, 256, 0, st>>>(-alpha, p.as<double>(), 1.0, r2.as<double>(), nz);        // r2 -= a p
    GF_CHECK_LAUNCH();
    C.rmv(r1.as<double>(), s.as<double>());                   // s = A' r1 + r2
    axpby_kernel<<<gz, 256, 0, st>>>(1.0, r2.as<double>(), 1.0, s.as<double>(), nz);
    GF_CHECK_LAUNCH();
    const double gnew = C.dot(s.as<double>(), s.as<double>(), nz, false);
    if (gnew <= thresh) return it;
    axpby_kernel<<<gz, 256, 0, st>>>(1.0, s.as<double>(), gnew / gamma, p.as<double>(), nz);   // p = s + b p
    GF_CHECK_LAUNCH();
    gamma = gnew;
  }
  *ok = false;
  return max_inner;
}

// project_indirect (projection.py:130-162): fp64 device vectors.
int64_t project_indirect_dev(const gf_matrix* A, bool tall, gf_comm* comm, const double* c, const double* d,
                             const double* xw, const double* yw, double tol, int64_t max_inner, double* x,
                             double* y, bool* ok, cudaStream_t st) {
  const int64_t m = A->m, n = A->n;
  int64_t it;
  if (tall) {
    if (xw) GF_CUDA(cudaMemcpyAsync(x, xw, n * 8, cudaMemcpyDeviceToDevice, st));
    else GF_CUDA(cudaMemsetAsync(x, 0, n * 8, st));
    it = cgls_solve(A, true, comm, d, c, x, tol, max_inner, ok, st);
    if (m > 0) matvec(A, false, x, y, st);
  } else {
    DBuf z(std::max<int64_t>(m, 1) * 8), negd(std::max<int64_t>(m, 1) * 8), t(n * 8);
    if (yw) sub_kernel<<<vblocks(m), 256, 0, st>>>(yw, d, z.as<double>(), m);   // z0 = y_warm - d
    else GF_CUDA(cudaMemsetAsync(z.p, 0, m * 8, st));
    GF_CUDA(cudaMemsetAsync(negd.p, 0, m * 8, st));
    sub_kernel<<<vblocks(m), 256, 0, st>>>(negd.as<double>(), d, negd.as<double>(), m);
    GF_CHECK_LAUNCH();
    it = cgls_solve(A, false, comm, c, negd.as<double>(), z.as<double>(), tol, max_inner, ok, st);
    // y = d + z ; x = c - A' z
    GF_CUDA(cudaMemcpyAsync(y, d, m * 8, cudaMemcpyDeviceToDevice, st));
    axpby_kernel<<<vblocks(m), 256, 0, st>>>(1.0, z.as<double>(), 1.0, y, m);
    matvec(A, true, z.as<double>(), t.as<double>(), st);
    sub_kernel<<<vblocks(n), 256, 0, st>>>(c, t.as<double>(), x, n);
    GF_CHECK_LAUNCH();
  }
  GF_CUDA(cudaStreamSynchronize(st));
  return it;
}

}  // namespace gf
