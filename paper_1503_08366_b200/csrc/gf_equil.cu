// Regularised Sinkhorn-Knopp equilibration (p = 2) and the even Frobenius
// rescale (reference equilibration.py:134-224, Alg. 2 of the paper).
//
// One sweep = a row pass  d_i = n / ((A∘A) e)_i + gamma/m)   (equilibration.py:176)
//           + a column pass e_j = m / ((A∘A)' d)_j + gamma/n) (equilibration.py:177)
// Both passes are HBM-bound streaming reductions over A in fp64 (A∘A is never
// materialised; the reference forms it in 256-row blocks).  Under a row
// partition the column sums and the ||d - d_prev||^2 partial are all-reduced,
// everything else is rank-local.

#include <vector>

#include "gf_internal.h"
#include "gf_gemv.cuh"

namespace gf {

// d_new_i = n_cols / (sum_j A_ij^2 w_j + reg); accumulates ||d_new - d_prev||^2,
// sum of row sums (all-zero check) and a bad-value count into part[block][3].
template <typename T>
__global__ void __launch_bounds__(kRowThreads)
sq_row_kernel(const T* __restrict__ A, int64_t rows, int64_t ld, int64_t n, const double* __restrict__ w,
              int mode, double numer, double reg, double* __restrict__ dout, const double* __restrict__ dprev,
              const double* __restrict__ dscale, double* __restrict__ part) {
  // mode 0: Sinkhorn row update (dout = numer / (rs + reg)); mode 1: Frobenius
  // partial sum_i dscale_i^2 * rs_i (no output vector); mode 2: dout = rs.
  // A warp takes two rows at a time: every weight w_j is loaded once for
  // both (the weight loads were as many as the matrix loads), eight 16-byte
  // matrix loads in flight per lane.  Each row's sum is formed in the same
  // lane order as one row at a time (same bits).
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nvec = ld / VN;
  double s_diff = 0.0, s_rows = 0.0, s_bad = 0.0;
  for (int64_t rp = (int64_t)blockIdx.x * kRowWarps + warp; 2 * rp < rows; rp += (int64_t)gridDim.x * kRowWarps) {
    const int64_t r0 = 2 * rp;
    const bool two = r0 + 1 < rows;
    const V* ar0 = reinterpret_cast<const V*>(A + r0 * ld);
    const V* ar1 = reinterpret_cast<const V*>(A + (two ? r0 + 1 : r0) * ld);
    double acc0 = 0.0, acc1 = 0.0;
    for (int64_t v = lane; v < nvec; v += 128) {   // four guarded 16-byte loads per row issued together
      V a0[4], a1[4];                              // (unguarded, ptxas scheduled them load-use-load)
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (v + 32 * u < nvec) {
          a0[u] = ld_stream(ar0 + v + 32 * u);
          a1[u] = ld_stream(ar1 + v + 32 * u);
        }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (v + 32 * u >= nvec) break;
#pragma unroll
        for (int i = 0; i < VN; ++i) {
          const int64_t j = (v + 32 * u) * VN + i;
          if (j < n) {
            const double wj = __ldg(w + j);
            const double x0 = (double)vget(a0[u], i), x1 = (double)vget(a1[u], i);
            acc0 = fma(x0 * x0, wj, acc0);
            acc1 = fma(x1 * x1, wj, acc1);
          }
        }
      }
    }
    acc0 = warp_sum(acc0);
    acc1 = warp_sum(acc1);
    if (lane == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && !two) break;
        const int64_t r = r0 + h;
        const double acc = h == 0 ? acc0 : acc1;
        if (mode == 2) {          // plain weighted row sums of squares: dout = (A o A) w
          dout[r] = acc;
          s_rows += acc;
        } else if (mode == 0) {
          const double dn = numer / (acc + reg);
          dout[r] = dn;
          if (dprev != nullptr) {
            const double df = dn - dprev[r];
            s_diff += df * df;
          }
          if (!(dn > 0.0) || !isfinite(dn)) s_bad += 1.0;
          s_rows += acc;
        } else {
          const double dr = dscale[r];
          s_rows += (dr * dr) * acc;
        }
      }
    }
  }
  __shared__ double sh[kRowWarps][3];
  if (lane == 0) { sh[warp][0] = s_diff; sh[warp][1] = s_rows; sh[warp][2] = s_bad; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int w2 = 0; w2 < kRowWarps; ++w2) s += sh[w2][threadIdx.x];
    part[blockIdx.x * 3 + threadIdx.x] = s;
  }
}

// e_new_j = numer / (c_j + reg); part[block][0..1] = ||e_new - e||^2, bad count.
__global__ void col_update_kernel(const double* __restrict__ c, int64_t n, double numer, double reg,
                                  double* __restrict__ e, double* __restrict__ part) {
  double s_diff = 0.0, s_bad = 0.0;
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double en = numer / (c[j] + reg);
    const double df = en - e[j];
    s_diff += df * df;
    if (!(en > 0.0) || !isfinite(en)) s_bad += 1.0;
    e[j] = en;
  }
  s_diff = warp_sum(s_diff);
  s_bad = warp_sum(s_bad);
  __shared__ double sh[8][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sh[warp][0] = s_diff; sh[warp][1] = s_bad; }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) s += sh[w][threadIdx.x];
    part[blockIdx.x * 2 + threadIdx.x] = s;
  }
}

// Deterministic sum of part[count][stride] columns -> out[stride] (one block).
__global__ void sum_parts(const double* __restrict__ part, int64_t count, int stride, double* __restrict__ out) {
  __shared__ double sh[256];
  for (int k = 0; k < stride; ++k) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) s += part[i * stride + k];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[k] = sh[0];
    __syncthreads();
  }
}

// out = sum_j a_j b_j, one CTA, fixed order
__global__ void fro2_dot_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += a[i] * b[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

__global__ void sqrt_inplace(double* x, int64_t n) {
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    x[j] = sqrt(x[j]);
}

__global__ void scal_inplace(double* x, int64_t n, const double* s, int inverse) {
  const double f = inverse ? 1.0 / *s : *s;
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    x[j] = inverse ? x[j] / *s : x[j] * f;
}

__global__ void fill_kernel(double* x, int64_t n, double v) {
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    x[j] = v;
}

__global__ void square_into(const double* x, double* y, int64_t n) {
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    y[j] = x[j] * x[j];
}

static unsigned vgrid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 1024)); }

static double global_rows(gf_matrix* A, gf_comm* comm, cudaStream_t st) {
  if (!comm_active(comm)) return (double)A->m;
  DBuf b(sizeof(double));
  double m = (double)A->m;
  GF_CUDA(cudaMemcpyAsync(b.p, &m, sizeof(double), cudaMemcpyHostToDevice, st));
  allreduce_sum(comm, b.as<double>(), 1, st);
  GF_CUDA(cudaMemcpyAsync(&m, b.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  return m;
}

template <typename T>
static EquilResult equil_t(gf_matrix* A, double gamma, double eps, int64_t max_iter, gf_comm* comm,
                           double* d_out, double* e_out, cudaStream_t st, SweepCb cb, void* user) {
  const int sms = num_sms();
  const int64_t m = A->m, n = A->n, ld = A->ld;
  const double mg = global_rows(A, comm, st);
  if (gamma < 0.0) gamma = (mg + (double)n) * sqrt(2.220446049250313e-16);  // (m+n)*sqrt(eps_fp64)
  if (!(eps > 0.0)) eps = 1e-4 * sqrt(std::max(mg, (double)n));
  const int64_t rgrid = row_grid(std::max<int64_t>(m, 1), sms);
  const ColPlan cp = plan_cols(std::max<int64_t>(m, 1), ld, Vec16<T>::n, sms);
  DBuf dA(std::max<int64_t>(m, 1) * sizeof(double)), dB(std::max<int64_t>(m, 1) * sizeof(double));
  DBuf rpart(rgrid * 3 * sizeof(double)), cpart((size_t)cp.slabs * ld * sizeof(double));
  DBuf csum((ld + 4) * sizeof(double)), epart(1024 * 2 * sizeof(double)), scal(8 * sizeof(double));
  double* e = e_out;  // device, n
  fill_kernel<<<vgrid(n), 256, 0, st>>>(e, n, 1.0);
  double* d_it = dA.as<double>();
  double* d_prev = dB.as<double>();
  bool have_prev = false, converged = false;
  int64_t k = 0;
  double h[4];
  while (k < max_iter) {
    ++k;
    if (m > 0) {
      sq_row_kernel<T><<<(unsigned)rgrid, kRowThreads, 0, st>>>((const T*)A->data, m, ld, n, e, 0, (double)n,
                                                                gamma / mg, d_it, have_prev ? d_prev : nullptr,
                                                                nullptr, rpart.as<double>());
      GF_CHECK_LAUNCH();
      sum_parts<<<1, 256, 0, st>>>(rpart.as<double>(), rgrid, 3, scal.as<double>());  // [ddiff, rowsum, bad]
      colgemv_kernel<T, 1, true><<<dim3((unsigned)cp.col_blocks, (unsigned)cp.slabs), kColThreads, 0, st>>>(
          (const T*)A->data, m, ld, d_it, d_it, cp.rows_per_slab, cpart.as<double>(), nullptr);
      GF_CHECK_LAUNCH();
      colreduce_kernel<<<dim3((unsigned)ceil_div(ld, 32), 1), dim3(32, 8), 0, st>>>(cpart.as<double>(), cp.slabs,
                                                                                    ld, 1, csum.as<double>(), nullptr);
      GF_CHECK_LAUNCH();
    } else {
      GF_CUDA(cudaMemsetAsync(scal.p, 0, 3 * sizeof(double), st));
      GF_CUDA(cudaMemsetAsync(csum.p, 0, ld * sizeof(double), st));
    }
    if (comm_active(comm)) {
      // [c (ld) | ddiff, rowsum, bad] reduced together
      GF_CUDA(cudaMemcpyAsync(csum.as<double>() + ld, scal.p, 3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
      allreduce_sum(comm, csum.as<double>(), ld + 3, st);
      GF_CUDA(cudaMemcpyAsync(scal.p, csum.as<double>() + ld, 3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    const unsigned eg = (unsigned)std::min<int64_t>(ceil_div(n, 256), 1024);
    col_update_kernel<<<eg, 256, 0, st>>>(csum.as<double>(), n, mg, gamma / (double)n, e, epart.as<double>());
    GF_CHECK_LAUNCH();
    sum_parts<<<1, 256, 0, st>>>(epart.as<double>(), eg, 2, scal.as<double>() + 3);  // [ediff, ebad]
    GF_CUDA(cudaMemcpyAsync(h, scal.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    double h2[2];
    GF_CUDA(cudaMemcpyAsync(h2, scal.as<double>() + 3, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    GF_CUDA(cudaStreamSynchronize(st));
    if (k == 1 && !(h[1] > 0.0))
      throw_error(GF_E_DEGENERATE_INPUT, "cannot equilibrate an all-zero matrix");
    if (cb != nullptr) {   // on_sweep(k, d_k^(1/p), e_k^(1/p)), before the convergence test
      std::vector<double> hd((size_t)std::max<int64_t>(m, 0)), he((size_t)n);
      if (m > 0) GF_CUDA(cudaMemcpyAsync(hd.data(), d_it, m * sizeof(double), cudaMemcpyDeviceToHost, st));
      GF_CUDA(cudaMemcpyAsync(he.data(), e, n * sizeof(double), cudaMemcpyDeviceToHost, st));
      GF_CUDA(cudaStreamSynchronize(st));
      for (auto& v : hd) v = sqrt(v);
      for (auto& v : he) v = sqrt(v);
      cb(k, hd.data(), he.data(), m, n, user);
    }
    const bool bad = h[2] > 0.0 || h2[1] > 0.0;
    if (bad) {
      throw_error(GF_E_NUMERIC,
                  "equilibration iterates are not finite; use gamma > 0 for matrices that cannot be equilibrated");
    }
    if (have_prev && sqrt(h2[0]) <= eps && sqrt(h[0]) <= eps) {
      converged = true;
      break;
    }
    std::swap(d_it, d_prev);
    have_prev = true;
  }
  // the last row update is in d_it unless we swapped after it
  const double* d_last = converged ? d_it : d_prev;
  if (m > 0) GF_CUDA(cudaMemcpyAsync(d_out, d_last, m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  // ||D A E||_F^2 = sum_i d_i sum_j a_ij^2 e_j = sum_j e_j csum_j (squared
  // scalings; csum: the last sweep's column sums, made with the final d) --
  // rescale_even's norm without another pass over A
  fro2_dot_kernel<<<1, 256, 0, st>>>(e, csum.as<double>(), n, scal.as<double>() + 5);
  sqrt_inplace<<<vgrid(m), 256, 0, st>>>(d_out, m);
  sqrt_inplace<<<vgrid(n), 256, 0, st>>>(e, n);
  GF_CHECK_LAUNCH();
  double fro2 = -1.0;
  GF_CUDA(cudaMemcpyAsync(&fro2, scal.as<double>() + 5, sizeof(double), cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  EquilResult r{k, converged, gamma};
  r.fro2 = fro2;
  return r;
}

EquilResult equilibrate(gf_matrix* A, double gamma, double eps, int64_t max_iter, gf_comm* comm, double* d_dev,
                        double* e_dev, cudaStream_t st, SweepCb cb, void* user) {
  GF_REQUIRE(max_iter >= 1, GF_E_PARAMETER, "max_iter must be at least 1");
  if (A->dtype == GF_F32) return equil_t<float>(A, gamma, eps, max_iter, comm, d_dev, e_dev, st, cb, user);
  return equil_t<double>(A, gamma, eps, max_iter, comm, d_dev, e_dev, st, cb, user);
}

static void apply_rescale(int64_t m, int64_t n, double mg, double fro2, double* d, double* e, cudaStream_t st);

template <typename T>
static void rescale_t(gf_matrix* A, double* d, double* e, gf_comm* comm, cudaStream_t st) {
  const int sms = num_sms();
  const int64_t m = A->m, n = A->n;
  const double mg = global_rows(A, comm, st);
  const int64_t rgrid = row_grid(std::max<int64_t>(m, 1), sms);
  DBuf e2(std::max<int64_t>(n, 1) * sizeof(double)), rpart(rgrid * 3 * sizeof(double)), scal(4 * sizeof(double));
  square_into<<<vgrid(n), 256, 0, st>>>(e, e2.as<double>(), n);
  GF_CUDA(cudaMemsetAsync(scal.p, 0, 4 * sizeof(double), st));
  if (m > 0) {
    sq_row_kernel<T><<<(unsigned)rgrid, kRowThreads, 0, st>>>((const T*)A->data, m, A->ld, n, e2.as<double>(), 1,
                                                              0.0, 0.0, nullptr, nullptr, d, rpart.as<double>());
    GF_CHECK_LAUNCH();
    sum_parts<<<1, 256, 0, st>>>(rpart.as<double>(), rgrid, 3, scal.as<double>());
  }
  if (comm_active(comm)) allreduce_sum(comm, scal.as<double>(), 3, st);
  double h[3];
  GF_CUDA(cudaMemcpyAsync(h, scal.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  apply_rescale(m, n, mg, h[1], d, e, st);
}

// d, e /= sqrt(||D A E||_F / sqrt(min(m, n))) (equilibration.py:214-224)
static void apply_rescale(int64_t m, int64_t n, double mg, double fro2, double* d, double* e, cudaStream_t st) {
  const double fro = sqrt(fro2);
  const double factor = fro / sqrt(std::min(mg, (double)n));
  if (!std::isfinite(factor) || factor == 0.0)
    throw_error(GF_E_DEGENERATE_INPUT, "scaled matrix has zero or non-finite norm");
  const double s = sqrt(factor);
  DBuf sv(sizeof(double));
  GF_CUDA(cudaMemcpyAsync(sv.p, &s, sizeof(double), cudaMemcpyHostToDevice, st));
  scal_inplace<<<vgrid(m), 256, 0, st>>>(d, m, sv.as<double>(), 1);
  scal_inplace<<<vgrid(n), 256, 0, st>>>(e, n, sv.as<double>(), 1);
  GF_CHECK_LAUNCH();
  GF_CUDA(cudaStreamSynchronize(st));
}

void rescale_even_fro2(gf_matrix* A, double* d, double* e, double fro2, gf_comm* comm, cudaStream_t st) {
  apply_rescale(A->m, A->n, global_rows(A, comm, st), fro2, d, e, st);
}

// y = (A o A) x (x: n) or (A o A)' x (x: m), fp64 device vectors: the p = 2
// |A|^p handles of equilibration.py:94-125 behind check_equilibrated and
// equilibration_objective.
template <typename T>
static void sq_matvec_t(const gf_matrix* A, bool transpose, const double* x, double* y, cudaStream_t st) {
  const int sms = num_sms();
  const int64_t m = A->m, n = A->n, ld = A->ld;
  if (!transpose) {
    const int64_t rgrid = row_grid(std::max<int64_t>(m, 1), sms);
    DBuf part((size_t)rgrid * 3 * sizeof(double));
    sq_row_kernel<T><<<(unsigned)rgrid, kRowThreads, 0, st>>>((const T*)A->data, m, ld, n, x, 2, 1.0, 0.0, y,
                                                              nullptr, nullptr, part.as<double>());
    GF_CHECK_LAUNCH();
    GF_CUDA(cudaStreamSynchronize(st));
    return;
  }
  const ColPlan cp = plan_cols(std::max<int64_t>(m, 1), ld, Vec16<T>::n, sms);
  DBuf cpart((size_t)cp.slabs * ld * sizeof(double)), out((size_t)ld * sizeof(double));
  colgemv_kernel<T, 1, true><<<dim3((unsigned)cp.col_blocks, (unsigned)cp.slabs), kColThreads, 0, st>>>(
      (const T*)A->data, m, ld, x, x, cp.rows_per_slab, cpart.as<double>(), nullptr);
  GF_CHECK_LAUNCH();
  colreduce_kernel<<<dim3((unsigned)ceil_div(ld, 32), 1), dim3(32, 8), 0, st>>>(cpart.as<double>(), cp.slabs, ld, 1,
                                                                              out.as<double>(), nullptr);
  GF_CHECK_LAUNCH();
  GF_CUDA(cudaMemcpyAsync(y, out.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  GF_CUDA(cudaStreamSynchronize(st));
}

void sq_matvec(const gf_matrix* A, bool transpose, const double* x, double* y, cudaStream_t st) {
  if (A->dtype == GF_F32) sq_matvec_t<float>(A, transpose, x, y, st);
  else sq_matvec_t<double>(A, transpose, x, y, st);
}

void rescale_even(gf_matrix* A, double* d, double* e, gf_comm* comm, cudaStream_t st) {
  if (A->dtype == GF_F32) rescale_t<float>(A, d, e, comm, st);
  else rescale_t<double>(A, d, e, comm, st);
}

}  // namespace gf
