// Matrix storage, upload, diagonal scaling and plain matvecs.
//
// problem.py:30-49 coerces A to a C-contiguous float64 array; solver.py:142-145
// materialises A_hat = (d[:,None] * A) * e[None,:] as a second array.  Here A
// is uploaded once into library memory in the working dtype with a 128-byte
// padded row stride, and scaled IN PLACE into A_hat: the solve never needs the
// unscaled A again because the residuals are taken through A_hat with the
// diagonal scalings folded in (A x = D^-1 A_hat E^-1 x).

#include <mutex>
#include <cstring>
#include "gf_internal.h"
#include "gf_gemv.cuh"

namespace gf {

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

void copy_in(double* dst_dev, const double* src, int64_t n, cudaStream_t st) {
  if (n > 0) GF_CUDA(cudaMemcpyAsync(dst_dev, src, n * sizeof(double), cudaMemcpyDefault, st));
}
void copy_out(double* dst, const double* src_dev, int64_t n, cudaStream_t st) {
  if (n > 0) GF_CUDA(cudaMemcpyAsync(dst, src_dev, n * sizeof(double), cudaMemcpyDefault, st));
}

template <typename TS, typename TD>
__global__ void convert_rows(const TS* __restrict__ src, int64_t lds, TD* __restrict__ dst, int64_t ldd,
                             int64_t rows, int64_t cols) {
  const int64_t r = blockIdx.y;
  if (r >= rows) return;
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < ldd; j += (int64_t)gridDim.x * blockDim.x)
    dst[r * ldd + j] = j < cols ? (TD)src[r * lds + j] : (TD)0;
}

template <typename TS, typename TD>
static void launch_convert(const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols,
                           cudaStream_t st) {
  for (int64_t r0 = 0; r0 < rows; r0 += 65535) {
    const int64_t nr = std::min<int64_t>(65535, rows - r0);
    dim3 grid((unsigned)std::min<int64_t>(ceil_div(ldd, 256), 32), (unsigned)nr);
    convert_rows<TS, TD><<<grid, 256, 0, st>>>((const TS*)src + r0 * lds, lds, (TD*)dst + r0 * ldd, ldd, nr, cols);
    GF_CHECK_LAUNCH();
  }
}

static void convert_any(int sdt, const void* src, int64_t lds, int ddt, void* dst, int64_t ldd, int64_t rows,
                        int64_t cols, cudaStream_t st) {
  if (sdt == GF_F64 && ddt == GF_F64) launch_convert<double, double>(src, lds, dst, ldd, rows, cols, st);
  else if (sdt == GF_F64 && ddt == GF_F32) launch_convert<double, float>(src, lds, dst, ldd, rows, cols, st);
  else if (sdt == GF_F32 && ddt == GF_F64) launch_convert<float, double>(src, lds, dst, ldd, rows, cols, st);
  else launch_convert<float, float>(src, lds, dst, ldd, rows, cols, st);
}

static bool is_pinned_host_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Pinned staging buffers for pageable host sources, kept for the process.
struct Staging {
  std::mutex mu;
  static constexpr int kBufs = 3;
  static constexpr size_t kBytes = (size_t)96 << 20;
  char* buf[kBufs] = {nullptr, nullptr, nullptr};
  cudaEvent_t done[kBufs] = {nullptr, nullptr, nullptr};
};
static Staging& staging() {
  static Staging s;
  return s;
}

// A pageable host matrix (a plain numpy array -- what a reference user
// passes) moves through cudaMemcpy at ~10 GB/s: the driver bounces it
// through a small pinned buffer.  Here host threads (OpenMP) copy row chunks
// into three pinned 96 MB buffers that the copy engine drains asynchronously,
// so the host copy of chunk i overlaps the DMA of chunks i-1, i-2.
static void upload_pageable(gf_matrix* M, const void* src, int src_dtype, int64_t src_ld, cudaStream_t st) {
  const size_t ses = src_dtype == GF_F32 ? 4 : 8;
  const size_t row_src = (size_t)M->n * ses;
  Staging& S = staging();
  std::lock_guard<std::mutex> lk(S.mu);
  for (int b = 0; b < Staging::kBufs; ++b)
    if (S.buf[b] == nullptr) {
      GF_CUDA(cudaMallocHost(&S.buf[b], Staging::kBytes));
      GF_CUDA(cudaEventCreateWithFlags(&S.done[b], cudaEventDisableTiming));
    }
  const int64_t rows_per = std::max<int64_t>(1, (int64_t)(Staging::kBytes / std::max<size_t>(row_src, 1)));
  DBuf dstage;
  if (src_dtype != M->dtype) dstage.alloc((size_t)std::min(rows_per, M->m) * row_src);
  bool used[Staging::kBufs] = {false, false, false};
  int b = 0;
  for (int64_t r0 = 0; r0 < M->m; r0 += rows_per, b = (b + 1) % Staging::kBufs) {
    const int64_t nr = std::min(rows_per, M->m - r0);
    if (used[b]) GF_CUDA(cudaEventSynchronize(S.done[b]));   // its previous DMA has drained
    char* dst = S.buf[b];
    const char* sp = (const char*)src + (size_t)r0 * src_ld * ses;
    const size_t total = (size_t)nr * row_src;
    if ((size_t)src_ld * ses == row_src) {   // contiguous rows: one flat parallel copy
      const int64_t parts = 64;
#pragma omp parallel for schedule(static)
      for (int64_t q = 0; q < parts; ++q) {
        const size_t a = total * q / parts, e = total * (q + 1) / parts;
        memcpy(dst + a, sp + a, e - a);
      }
    } else {
#pragma omp parallel for schedule(static)
      for (int64_t r = 0; r < nr; ++r) memcpy(dst + r * row_src, sp + (size_t)r * src_ld * ses, row_src);
    }
    if (src_dtype == M->dtype) {
      GF_CUDA(cudaMemcpy2DAsync((char*)M->data + (size_t)r0 * M->ld * M->esize(), M->ld * M->esize(), dst, row_src,
                                row_src, nr, cudaMemcpyHostToDevice, st));
    } else {
      GF_CUDA(cudaMemcpyAsync(dstage.p, dst, total, cudaMemcpyHostToDevice, st));
      convert_any(src_dtype, dstage.p, M->n, M->dtype, (char*)M->data + (size_t)r0 * M->ld * M->esize(), M->ld,
                  nr, M->n, st);
    }
    GF_CUDA(cudaEventRecord(S.done[b], st));
    used[b] = true;
  }
  GF_CUDA(cudaStreamSynchronize(st));
}

void matrix_upload(gf_matrix* M, const void* src, int src_dtype, int64_t src_ld, cudaStream_t st) {
  const size_t ses = src_dtype == GF_F32 ? 4 : 8;
  if (M->m == 0) return;
  if (is_device_ptr(src)) {
    convert_any(src_dtype, src, src_ld, M->dtype, M->data, M->ld, M->m, M->n, st);
    return;
  }
  if (!is_pinned_host_ptr(src) && (size_t)M->m * M->n * ses >= ((size_t)64 << 20)) {
    if (M->ld > M->n) GF_CUDA(cudaMemsetAsync(M->data, 0, (size_t)M->m * M->ld * M->esize(), st));
    upload_pageable(M, src, src_dtype, src_ld, st);
    return;
  }
  if (src_dtype == M->dtype) {
    // host -> device with the padding columns zeroed
    GF_CUDA(cudaMemsetAsync(M->data, 0, (size_t)M->m * M->ld * M->esize(), st));
    GF_CUDA(cudaMemcpy2DAsync(M->data, M->ld * M->esize(), src, src_ld * ses, M->n * ses, M->m,
                              cudaMemcpyHostToDevice, st));
    return;
  }
  // dtype change: stage row blocks of the host matrix on the device, convert
  const int64_t rows_per = std::max<int64_t>(1, ((int64_t)256 << 20) / std::max<int64_t>(1, M->n * (int64_t)ses));
  DBuf stage((size_t)std::min(rows_per, M->m) * M->n * ses);
  for (int64_t r0 = 0; r0 < M->m; r0 += rows_per) {
    const int64_t nr = std::min(rows_per, M->m - r0);
    GF_CUDA(cudaMemcpy2DAsync(stage.p, M->n * ses, (const char*)src + r0 * src_ld * ses, src_ld * ses,
                              M->n * ses, nr, cudaMemcpyHostToDevice, st));
    convert_any(src_dtype, stage.p, M->n, M->dtype, (char*)M->data + r0 * M->ld * M->esize(), M->ld, nr, M->n, st);
  }
  GF_CUDA(cudaStreamSynchronize(st));
}

void matrix_to_f64(const gf_matrix* M, double* dst, cudaStream_t st) {
  convert_any(M->dtype, M->data, M->ld, GF_F64, dst, M->n, M->m, M->n, st);
}

// A_ij <- (d_i * A_ij) * e_j in fp64, rounded to the working dtype
// (solver.py:145 evaluation order).
template <typename T>
__device__ __forceinline__ T scale1(T a, double dr, double ej) {
  return (T)((dr * (double)a) * ej);
}

// One CTA per row (grid-stride), 16-byte vectors: A is read and written
// once (2 m n s bytes); columns past n are the zero padding and stay zero.
// With `amax` set, max |A_hat| over the real columns is accumulated as float
// bits (non-negative floats order like their bits) for the Gram's fp16 split
// scale, saving it a pass over A_hat.
template <typename T>
__global__ void __launch_bounds__(256) scale_kernel(T* __restrict__ A, int64_t rows, int64_t ld, int64_t n,
                                                    const double* __restrict__ d, const double* __restrict__ e,
                                                    unsigned* __restrict__ amax) {
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
  const int64_t nv = (n + VN - 1) / VN;
  float mx = 0.0f;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const double dr = d[r];
    V* row = reinterpret_cast<V*>(A + r * ld);
    // four vectors per thread loaded before any is written back (each element
    // is read and written by the same thread): four 16-byte loads in flight
    for (int64_t v0 = threadIdx.x; v0 < nv; v0 += 4 * (int64_t)blockDim.x) {
      V a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t v = v0 + u * (int64_t)blockDim.x;
        if (v < nv) a[u] = row[v];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t v = v0 + u * (int64_t)blockDim.x;
        if (v >= nv) break;
        const int64_t j = v * VN;
        if constexpr (VN == 4) {
          a[u].x = scale1(a[u].x, dr, e[j]);
          if (j + 1 < n) a[u].y = scale1(a[u].y, dr, e[j + 1]);
          if (j + 2 < n) a[u].z = scale1(a[u].z, dr, e[j + 2]);
          if (j + 3 < n) a[u].w = scale1(a[u].w, dr, e[j + 3]);
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf((float)a[u].x), fabsf((float)a[u].y)),
                               fmaxf(fabsf((float)a[u].z), fabsf((float)a[u].w))));
        } else {
          a[u].x = scale1(a[u].x, dr, e[j]);
          if (j + 1 < n) a[u].y = scale1(a[u].y, dr, e[j + 1]);
          mx = fmaxf(mx, fmaxf(fabsf((float)a[u].x), fabsf((float)a[u].y)));
        }
        row[v] = a[u];
      }
    }
  }
  if (amax != nullptr) {   // (padding lanes hold zeros: they do not raise the max)
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(amax, __float_as_uint(mx));
  }
}

void scale_matrix(gf_matrix* M, const double* d, const double* e, cudaStream_t st, unsigned* amax) {
  if (M->m == 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(M->m, (int64_t)num_sms() * 8);
  if (M->dtype == GF_F32) scale_kernel<float><<<grid, 256, 0, st>>>((float*)M->data, M->m, M->ld, M->n, d, e, amax);
  else scale_kernel<double><<<grid, 256, 0, st>>>((double*)M->data, M->m, M->ld, M->n, d, e, amax);
  GF_CHECK_LAUNCH();
}

__global__ void colreduce_kernel(const double* __restrict__ part, int64_t slabs, int64_t ld, int nrhs,
                                 double* __restrict__ out, const int* __restrict__ status) {
  if (status != nullptr && *status != 0) return;
  __shared__ double sh[8][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t j = (int64_t)blockIdx.x * 32 + tx;
  const int k = blockIdx.y;
  double s = 0.0;
  if (j < ld)
    for (int64_t sl = ty; sl < slabs; sl += 8) s += part[(sl * nrhs + k) * ld + j];
  sh[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && j < ld) {
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += sh[i][tx];
    out[k * ld + j] = t;
  }
}

struct StoreEpi {
  static constexpr int NR = 0;
  double* y;
  __device__ bool active() const { return true; }
  __device__ void row(int64_t r, const double* dots, double*, unsigned&) const { y[r] = dots[0]; }
};

template <typename T>
__global__ void to_padded(const double* __restrict__ x, int64_t n, T* __restrict__ out, int64_t ld) {
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < ld; j += (int64_t)gridDim.x * blockDim.x)
    out[j] = j < n ? (T)x[j] : (T)0;
}

template <typename T>
static void matvec_t(const gf_matrix* A, bool transpose, const double* x, double* y, cudaStream_t st) {
  const int sms = num_sms();
  if (!transpose) {
    DBuf xp(A->ld * sizeof(T));
    to_padded<T><<<(unsigned)std::min<int64_t>(ceil_div(A->ld, 256), 1024), 256, 0, st>>>(x, A->n, xp.as<T>(), A->ld);
    GF_CHECK_LAUNCH();
    StoreEpi epi{y};
    rowgemv_kernel<T, 1, StoreEpi><<<(unsigned)row_grid(A->m, sms), kRowThreads, 0, st>>>(
        (const T*)A->data, A->m, A->ld, xp.as<T>(), xp.as<T>(), epi, nullptr);
    GF_CHECK_LAUNCH();
    GF_CUDA(cudaStreamSynchronize(st));
    return;
  }
  const ColPlan p = plan_cols(A->m, A->ld, Vec16<T>::n, sms);
  DBuf part((size_t)p.slabs * A->ld * sizeof(double));
  DBuf out((size_t)A->ld * sizeof(double));
  colgemv_kernel<T, 1, false><<<dim3((unsigned)p.col_blocks, (unsigned)p.slabs), kColThreads, 0, st>>>(
      (const T*)A->data, A->m, A->ld, x, x, p.rows_per_slab, part.as<double>(), nullptr);
  GF_CHECK_LAUNCH();
  colreduce_kernel<<<dim3((unsigned)ceil_div(A->ld, 32), 1), dim3(32, 8), 0, st>>>(part.as<double>(), p.slabs,
                                                                                  A->ld, 1, out.as<double>(), nullptr);
  GF_CHECK_LAUNCH();
  GF_CUDA(cudaMemcpyAsync(y, out.p, A->n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  GF_CUDA(cudaStreamSynchronize(st));
}

void matvec(const gf_matrix* A, bool transpose, const double* x, double* y, cudaStream_t st) {
  if (A->dtype == GF_F32) matvec_t<float>(A, transpose, x, y, st);
  else matvec_t<double>(A, transpose, x, y, st);
}

}  // namespace gf
