// Streaming matrix-vector kernels over row-major, 128-byte-padded matrices.
//
//  rowgemv : y_r = <A_r, x_k> for 1-2 right-hand sides, one warp per row,
//            16-byte vector loads of A (L1 no-allocate: A is read once per
//            pass) and of x (L1/L2 resident), 4-8 loads in flight per lane;
//            the per-row results go to an epilogue functor, run for 32 rows
//            at a time on the warp's lanes, whose reduction scalars are
//            folded per CTA into `part`.
//  colgemv : partial column sums  part[slab][k][j] = sum_{r in slab} f(A_rj) w_k[r]
//            for 1-2 weight vectors; a CTA owns a 256-vector column strip of
//            one row slab, so every warp load is a contiguous 512 B segment;
//            fp64 accumulation; a second, deterministic pass sums the slabs.
//
// Both are HBM-bound (arithmetic intensity <= 0.5 flop/byte); their roofline is
// the copy bandwidth in MEASURED_PEAKS.json.
#pragma once

#include "gf_common.cuh"

namespace gf {

constexpr int kRowThreads = 256;
constexpr int kRowWarps = kRowThreads / kWarp;

template <typename V>
__device__ __forceinline__ V ldg_vec(const V* p) { return __ldg(p); }

// Epi interface:
//   static constexpr int NR;                        reduction scalars per row
//   __device__ bool active() const;                 false -> kernel returns
//   __device__ void row(int64_t r, const double* dots, double* red, unsigned& flags) const;
template <typename T, int NRHS, class Epi>
__global__ void __launch_bounds__(kRowThreads)
rowgemv_kernel(const T* __restrict__ A, int64_t rows, int64_t ld, const T* __restrict__ x0,
               const T* __restrict__ x1, Epi epi, double* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  if (!epi.active()) return;
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
  constexpr int NR = Epi::NR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nvec = ld / VN;
  const V* xv0 = reinterpret_cast<const V*>(x0);
  const V* xv1 = reinterpret_cast<const V*>(NRHS > 1 ? x1 : x0);
  double red[NR > 0 ? NR : 1];
#pragma unroll
  for (int k = 0; k < (NR > 0 ? NR : 1); ++k) red[k] = 0.0;
  unsigned flags = 0;
  // Rows r = w, w + W, ... (W warps in the grid) in batches of 32: the dot
  // products of a batch first, lane t keeping row t's; then the 32 epilogues
  // run in parallel on the lanes (a serial fp64 epilogue -- e.g. the
  // logistic prox's Newton loop -- is paid once per batch, not per row).
  const int64_t stride = (int64_t)gridDim.x * kRowWarps;
  for (int64_t rb = (int64_t)blockIdx.x * kRowWarps + warp; rb < rows; rb += 32 * stride) {
    double my0 = 0.0, my1 = 0.0;
    int cnt = 0;
    for (int t = 0; t < 32; ++t) {
      const int64_t r = rb + t * stride;
      if (r >= rows) break;
      ++cnt;
      const V* ar = reinterpret_cast<const V*>(A + r * ld);
      T s0 = 0, s1 = 0;
      int64_t v = lane;
      // one right-hand side: 8 row loads in flight per lane
      constexpr int U = NRHS > 1 ? 4 : 8;
      for (; v + (U - 1) * 32 < nvec; v += U * 32) {
        V a[U], b0[U], b1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          a[u] = ld_stream(ar + v + 32 * u);
          b0[u] = ldg_vec(xv0 + v + 32 * u);
          if (NRHS > 1) b1[u] = ldg_vec(xv1 + v + 32 * u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < VN; ++i) {
            s0 = fma(vget(a[u], i), vget(b0[u], i), s0);
            if (NRHS > 1) s1 = fma(vget(a[u], i), vget(b1[u], i), s1);
          }
      }
      for (; v < nvec; v += 32) {
        const V a = ld_stream(ar + v);
        const V b0 = ldg_vec(xv0 + v);
#pragma unroll
        for (int i = 0; i < VN; ++i) s0 = fma(vget(a, i), vget(b0, i), s0);
        if (NRHS > 1) {
          const V b1 = ldg_vec(xv1 + v);
#pragma unroll
          for (int i = 0; i < VN; ++i) s1 = fma(vget(a, i), vget(b1, i), s1);
        }
      }
      s0 = warp_sum(s0);
      if (NRHS > 1) s1 = warp_sum(s1);
      if (lane == t) { my0 = (double)s0; my1 = (double)s1; }
    }
    if (lane < cnt) {
      double dots[2] = {my0, my1};
      epi.row(rb + lane * stride, dots, red, flags);
    }
  }
#pragma unroll
  for (int k = 0; k < NR; ++k) red[k] = warp_sum(red[k]);
  flags = warp_or(flags);
  if (part == nullptr) return;
  __shared__ double sred[kRowWarps][NR + 1];
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NR; ++k) sred[warp][k] = red[k];
    sred[warp][NR] = (double)flags;
  }
  __syncthreads();
  if (threadIdx.x <= NR) {
    const int k = threadIdx.x;
    if (k < NR) {
      double s = 0.0;
      for (int w = 0; w < kRowWarps; ++w) s += sred[w][k];
      part[blockIdx.x * (NR + 1) + k] = s;
    } else {
      unsigned f = 0;
      for (int w = 0; w < kRowWarps; ++w) f |= (unsigned)sred[w][NR];
      part[blockIdx.x * (NR + 1) + NR] = (double)f;
    }
  }
}

constexpr int kColThreads = 256;

// part layout: [slab][k][ld]; SQ: use A_rj^2 (equilibration) instead of A_rj.
template <typename T, int NRHS, bool SQ>
__global__ void __launch_bounds__(kColThreads, 4)   // plan_cols sizes the grid for 4 CTAs/SM
colgemv_kernel(const T* __restrict__ A, int64_t rows, int64_t ld, const double* __restrict__ w0,
               const double* __restrict__ w1, int64_t rows_per_slab, double* __restrict__ part,
               const int* __restrict__ status) {
  if (status != nullptr && *status != 0) return;
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
  const int64_t cv = (int64_t)blockIdx.x * kColThreads + threadIdx.x;
  const int64_t nvec = ld / VN;
  const int64_t slab = blockIdx.y;
  const int64_t r0 = slab * rows_per_slab;
  const int64_t r1 = min(rows, r0 + rows_per_slab);
  double acc0[VN], acc1[VN];
#pragma unroll
  for (int i = 0; i < VN; ++i) { acc0[i] = 0.0; acc1[i] = 0.0; }
  if (cv < nvec) {
    const V* base = reinterpret_cast<const V*>(A) + cv;
    // U rows per step, every load issued before the first FMA (guarded loads
    // like the scaling pass; unguarded ones were scheduled load-use-load);
    // rows are accumulated in order, so the result does not depend on U
    constexpr int U = 4;
    for (int64_t r = r0; r < r1; r += U) {
      V a[U];
      double u0[U], u1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (r + u < r1) {
          a[u] = ld_stream(base + (r + u) * nvec);
          u0[u] = __ldg(w0 + r + u);
          if (NRHS > 1) u1[u] = __ldg(w1 + r + u);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (r + u >= r1) break;
#pragma unroll
        for (int i = 0; i < VN; ++i) {
          double x = (double)vget(a[u], i);
          if (SQ) x = x * x;
          acc0[i] = fma(x, u0[u], acc0[i]);
          if (NRHS > 1) acc1[i] = fma(x, u1[u], acc1[i]);
        }
      }
    }
    double* p0 = part + (slab * NRHS) * ld + cv * VN;
#pragma unroll
    for (int i = 0; i < VN; ++i) p0[i] = acc0[i];
    if (NRHS > 1) {
      double* p1 = part + (slab * NRHS + 1) * ld + cv * VN;
#pragma unroll
      for (int i = 0; i < VN; ++i) p1[i] = acc1[i];
    }
  }
}

// out[k][j] = sum_s part[s][k][j] for j < ld, fixed summation order.
// Block (32 columns x 8 slab lanes); grid x = ceil(ld / 32), y = NRHS.
__global__ void colreduce_kernel(const double* __restrict__ part, int64_t slabs, int64_t ld,
                                 int nrhs, double* __restrict__ out, const int* __restrict__ status);

struct ColPlan {
  int64_t slabs = 1, rows_per_slab = 1, col_blocks = 1;
};

inline ColPlan plan_cols(int64_t rows, int64_t ld, int vn, int sms) {
  ColPlan p;
  const int64_t nvec = ld / vn;
  p.col_blocks = ceil_div(nvec, kColThreads);
  // about 4 CTAs per SM (what the registers allow: 1024 threads x 4 rows of
  // 16-byte loads in flight, ~64 KB per SM -- with 2 per SM the pass ran at
  // 2.8 TB/s), and at least 64 rows per slab
  int64_t want = std::max<int64_t>(1, (int64_t)4 * sms / p.col_blocks);
  want = std::min<int64_t>(want, std::max<int64_t>(1, rows / 64));
  want = std::min<int64_t>(want, 4096);
  p.rows_per_slab = ceil_div(std::max<int64_t>(rows, 1), want);
  p.slabs = ceil_div(std::max<int64_t>(rows, 1), p.rows_per_slab);
  return p;
}

inline int64_t row_grid(int64_t rows, int sms) {
  return std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, kRowWarps), (int64_t)sms * 4));
}

}  // namespace gf
