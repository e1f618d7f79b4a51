// Dense setup kernels: Gram matrix, blocked Cholesky, triangular inverse.
//
// Reference: projection.py:86-94 forms G = A'A + I (tall) or AA' + I (wide)
// with dgemm and factors it with LAPACK potrf (scipy cho_factor); every
// projection then runs potrs.  Here the factor is computed once on the GPU in
// fp64 (blocked right-looking Cholesky: diagonal POTRF in shared memory, panel
// TRSM, trailing SYRK update as a tiled GEMM), inverted blockwise
// (recursive-doubling TRTRI: W21 = -W22 L21 W11) and assembled into
// G^-1 = W' W.  The per-iteration projection is then one coalesced GEMV over
// G^-1 (gf_solver.cu) instead of two latency-bound triangular solves; the bytes
// per iteration are the same (q^2) and lambda_min(G) >= 1 keeps the explicit
// inverse well conditioned.
//
// All factorization arithmetic is fp64 on the CUDA cores: B200's fp64 tensor
// and vector peaks are the same order, and the factor is O(q^3) against the
// O(m q^2) Gram.  The Gram itself reads the working-dtype matrix and
// accumulates in fp64.

#include <type_traits>
#include <vector>

#include <mutex>

#include "gf_internal.h"

namespace gf {

// ------------------------------------------------------------- tiled GEMM --
// C[i][j] = alpha * sum_k opA(i,k) opB(k,j) + beta * C[i][j]
//   opA(i,k) = AT ? A[k*lda + i] : A[i*lda + k]
//   opB(k,j) = BT ? B[j*ldb + k] : B[k*ldb + j]
// 64x64 output tile per 256-thread CTA, 16-deep K slices staged in shared
// memory, 4x4 fp64 accumulators per thread.  lower_only skips tiles strictly
// above the diagonal (symmetric outputs).  blockIdx.z indexes a batch.
constexpr int GB = 64, GK = 16;

template <typename TA, typename TB, bool AT, bool BT>
__global__ void __launch_bounds__(256) gemm_kernel(int64_t M, int64_t N, int64_t K, double alpha,
                                                   const TA* __restrict__ A, int64_t lda, int64_t sA,
                                                   const TB* __restrict__ B, int64_t ldb, int64_t sB,
                                                   double beta, double* __restrict__ C, int64_t ldc,
                                                   int64_t sC, int lower_only) {
  const int64_t ti = blockIdx.y, tj = blockIdx.x;
  if (lower_only && tj > ti) return;
  A += blockIdx.z * sA;
  B += blockIdx.z * sB;
  C += blockIdx.z * sC;
  __shared__ double As[GK][GB + 1];
  __shared__ double Bs[GK][GB + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t i0 = ti * GB, j0 = tj * GB;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  for (int64_t k0 = 0; k0 < K; k0 += GK) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      int ii, kk;
      if (AT) { ii = tid & 63; kk = (tid >> 6) + 4 * s; }
      else    { kk = tid & 15; ii = (tid >> 4) + 16 * s; }
      const int64_t gi = i0 + ii, gk = k0 + kk;
      double v = 0.0;
      if (gi < M && gk < K) v = (double)(AT ? A[gk * lda + gi] : A[gi * lda + gk]);
      As[kk][ii] = v;
      int jj, kb;
      if (BT) { kb = tid & 15; jj = (tid >> 4) + 16 * s; }
      else    { jj = tid & 63; kb = (tid >> 6) + 4 * s; }
      const int64_t gj = j0 + jj, gkb = k0 + kb;
      double w = 0.0;
      if (gj < N && gkb < K) w = (double)(BT ? B[gj * ldb + gkb] : B[gkb * ldb + gj]);
      Bs[kb][jj] = w;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < GK; ++k) {
      double ra[4], rb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) ra[a] = As[k][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) rb[b] = Bs[k][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(ra[a], rb[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t gi = i0 + ty + 16 * a;
    if (gi >= M) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t gj = j0 + tx + 16 * b;
      if (gj >= N) continue;
      double* c = C + gi * ldc + gj;
      *c = beta == 0.0 ? alpha * acc[a][b] : alpha * acc[a][b] + beta * *c;
    }
  }
}

// ------------------------------------------------- fp64 tensor-core GEMM --
// The same contract for fp64 operands on B200's fp64 tensor cores
// (mma.sync m8n8k4 f64 -> DMMA): 128 x 64 output tile per 256-thread CTA
// (8 warps as 4 x 2, 32 x 32 per warp = 4 x 4 MMA tiles, 32 fp64
// accumulators per thread), 16-deep K slices staged in shared memory with a
// register prefetch of the next slice.  Shared rows are padded to 8 mod 16
// doubles so each fragment load (4 k-rows x 8 m/n-columns per warp) fills
// the 16 double-wide banks exactly twice.  Used for the fp64 Gram, the
// Cholesky trailing updates, TRTRI and W'W.
constexpr int TBM = 128, TBN = 64, TBK = 16, TPA = TBM + 8, TPB = TBN + 8;

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool AT, bool BT>
__global__ void __launch_bounds__(256) dgemm_tc_kernel(int64_t M, int64_t N, int64_t K, double alpha,
                                                       const double* __restrict__ A, int64_t lda, int64_t sA,
                                                       const double* __restrict__ B, int64_t ldb, int64_t sB,
                                                       double beta, double* __restrict__ C, int64_t ldc,
                                                       int64_t sC, int lower_only, int kmode) {
  const int64_t i0 = (int64_t)blockIdx.y * TBM, j0 = (int64_t)blockIdx.x * TBN;
  if (lower_only && j0 > i0 + TBM - 1) return;
  // Triangular operands (kmode, set by trtri / the W'W product): the K range
  // of this tile outside which every product has a zero factor -- skipped
  // whole TBK chunks only, so the non-zero terms are added in the same order
  // (results identical to the full range).
  //   1: B lower triangular (B[k][j] = 0 for k < j): k >= j0
  //   2: A lower triangular (A[i][k] = 0 for k > i): k < i0 + TBM
  //   3: A' with A lower triangular (A[k][i] = 0 for k < i): k >= i0
  const int64_t kbeg = kmode == 1 ? (j0 / TBK) * TBK : (kmode == 3 ? (i0 / TBK) * TBK : 0);
  const int64_t kend = kmode == 2 ? min(K, i0 + TBM) : K;
  A += blockIdx.z * sA;
  B += blockIdx.z * sB;
  C += blockIdx.z * sC;
  __shared__ __align__(16) double As[TBK][TPA];
  __shared__ __align__(16) double Bs[TBK][TPB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  double ra[8], rb[4];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int idx = s * 256 + tid;
      int ii, kk;
      if (AT) { kk = idx >> 7; ii = idx & 127; } else { kk = idx & 15; ii = idx >> 4; }
      const int64_t gi = i0 + ii, gk = k0 + kk;
      ra[s] = (gi < M && gk < K) ? (AT ? A[gk * lda + gi] : A[gi * lda + gk]) : 0.0;
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int idx = s * 256 + tid;
      int nn, kk;
      if (BT) { kk = idx & 15; nn = idx >> 4; } else { kk = idx >> 6; nn = idx & 63; }
      const int64_t gj = j0 + nn, gk = k0 + kk;
      rb[s] = (gj < N && gk < K) ? (BT ? B[gj * ldb + gk] : B[gk * ldb + gj]) : 0.0;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int idx = s * 256 + tid;
      int ii, kk;
      if (AT) { kk = idx >> 7; ii = idx & 127; } else { kk = idx & 15; ii = idx >> 4; }
      As[kk][ii] = ra[s];
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int idx = s * 256 + tid;
      int nn, kk;
      if (BT) { kk = idx & 15; nn = idx >> 4; } else { kk = idx >> 6; nn = idx & 63; }
      Bs[kk][nn] = rb[s];
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int fk = lane & 3, fr = lane >> 2;   // fragment k row, m/n column
  if (kbeg < kend) load(kbeg);
  for (int64_t k0 = kbeg; k0 < kend; k0 += TBK) {
    store();
    __syncthreads();
    if (k0 + TBK < kend) load(k0 + TBK);   // next slice in flight during the MMAs
#pragma unroll
    for (int ks = 0; ks < TBK / 4; ++ks) {
      double fa[4], fb[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        fa[t] = As[ks * 4 + fk][wm * 32 + t * 8 + fr];
        fb[t] = Bs[ks * 4 + fk][wn * 32 + t * 8 + fr];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t gi = i0 + wm * 32 + a * 8 + fr;
    if (gi >= M) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gj = j0 + wn * 32 + b * 8 + fk * 2 + h;
        if (gj >= N) continue;
        double* c = C + gi * ldc + gj;
        *c = beta == 0.0 ? alpha * acc[a][b][h] : alpha * acc[a][b][h] + beta * *c;
      }
  }
}

// ---------------------------------------- pipelined fp64 tensor-core GEMM --
// The DMMA GEMM above stages one 16-deep K slice with a register prefetch:
// at q = 20000 TRTRI and W'W ran at 19-25 TF/s, the slice's global latency
// exposed behind 64 DMMAs per warp.  This one streams K slices through a
// PST-stage cp.async ring (16-byte copies, zero-filled past M / N / K) into
// 128 x 128 tiles: 8 warps as 2 x 4, a 64 x 32 warp tile = 8 x 4 DMMA.8x8x4
// tiles, 64 fp64 accumulators per thread, 12 fragment loads per 32 DMMAs.
// Every operand is staged in its global orientation -- k-contiguous rows
// [mn][k] (stride PKC = 20 doubles, 4 mod 16) or mn-contiguous rows [k][mn]
// (stride PMC = 136, 8 mod 16) -- both of which serve the m8n8k4 fragment
// pattern (8 mn x 4 k per warp) in the minimum two wavefronts.  The DMMA
// sequence over k (k4 steps in increasing order, the same kbeg / kend) is
// the old kernel's, so the two produce identical results.
constexpr int PBM = 128, PBK = 16, PST = 4, PMC = PBM + 8, PKC = PBK + 4;
constexpr int PSTAGE = PBM * PKC > PBK * PMC ? PBM * PKC : PBK * PMC;   // doubles per operand stage
constexpr size_t kPipeSmem = (size_t)PST * 2 * PSTAGE * sizeof(double);

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

// one PBM x PBK operand stage: KC = rows of the tile contiguous in k
// (X[mn * ld + k]), else contiguous in mn (X[k * ld + mn])
template <bool KC>
__device__ __forceinline__ void pipe_stage(double* S, const double* __restrict__ X, int64_t ld, int64_t mn0,
                                           int64_t MN, int64_t k0, int64_t K, int tid) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int c = s * 256 + tid;
    int r, e;   // stage row, element
    int64_t mn, k;
    if (KC) { r = c >> 3; e = (c & 7) * 2; mn = mn0 + r; k = k0 + e; }
    else { r = c >> 6; e = (c & 63) * 2; k = k0 + r; mn = mn0 + e; }
    int valid = 0;
    if (mn < MN && k < K) valid = KC ? (K - k >= 2 ? 2 : 1) : (MN - mn >= 2 ? 2 : 1);
    const double* src = valid ? (KC ? X + mn * ld + k : X + k * ld + mn) : X;
    cp_async16(S + (KC ? r * PKC + e : r * PMC + e), src, valid * 8);
  }
}

template <bool AT, bool BT>
__global__ void __launch_bounds__(256, 1) dgemm_pipe_kernel(int64_t M, int64_t N, int64_t K, double alpha,
                                                            const double* __restrict__ A, int64_t lda, int64_t sA,
                                                            const double* __restrict__ B, int64_t ldb, int64_t sB,
                                                            double beta, double* __restrict__ C, int64_t ldc,
                                                            int64_t sC, int lower_only, int kmode) {
  constexpr bool AKC = !AT, BKC = BT;   // A[i*lda+k] is k-contiguous; B[j*ldb+k] (BT) too
  const int64_t i0 = (int64_t)blockIdx.y * PBM, j0 = (int64_t)blockIdx.x * PBM;
  if (lower_only && j0 > i0 + PBM - 1) return;
  // kmode as in dgemm_tc_kernel, in TBK (16) units: the same DMMA sequence
  const int64_t kbeg = kmode == 1 ? (j0 / TBK) * TBK : (kmode == 3 ? (i0 / TBK) * TBK : 0);
  const int64_t kend = kmode == 2 ? min(K, i0 + PBM) : K;
  A += blockIdx.z * sA;
  B += blockIdx.z * sB;
  C += blockIdx.z * sC;
  extern __shared__ __align__(16) double psm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int fk = lane & 3, fr = lane >> 2;
  const int64_t nk = kend > kbeg ? (kend - kbeg + PBK - 1) / PBK : 0;
  auto SA = [&](int64_t s) { return psm + (size_t)(s % PST) * 2 * PSTAGE; };
  auto SB = [&](int64_t s) { return psm + (size_t)(s % PST) * 2 * PSTAGE + PSTAGE; };
#pragma unroll
  for (int s = 0; s < PST - 1; ++s) {
    if (s < nk) {
      pipe_stage<AKC>(SA(s), A, lda, i0, M, kbeg + s * PBK, K, tid);
      pipe_stage<BKC>(SB(s), B, ldb, j0, N, kbeg + s * PBK, K, tid);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int64_t it = 0; it < nk; ++it) {
    asm volatile("cp.async.wait_group %0;" ::"n"(PST - 2) : "memory");
    __syncthreads();   // stage it landed for every thread; stage it - 1 is free
    const int64_t nx = it + PST - 1;
    if (nx < nk) {
      pipe_stage<AKC>(SA(nx), A, lda, i0, M, kbeg + nx * PBK, K, tid);
      pipe_stage<BKC>(SB(nx), B, ldb, j0, N, kbeg + nx * PBK, K, tid);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    const double* sa = SA(it);
    const double* sb = SB(it);
#pragma unroll
    for (int ks = 0; ks < PBK / 4; ++ks) {
      const int k = ks * 4 + fk;
      double fa[8], fb[4];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int m = wm * 64 + t * 8 + fr;
        fa[t] = AKC ? sa[m * PKC + k] : sa[k * PMC + m];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int n = wn * 32 + u * 8 + fr;
        fb[u] = BKC ? sb[n * PKC + k] : sb[k * PMC + n];
      }
#pragma unroll
      for (int t = 0; t < 8; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma884(acc[t][u][0], acc[t][u][1], fa[t], fb[u]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int64_t gi = i0 + wm * 64 + t * 8 + fr;
    if (gi >= M) continue;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gj = j0 + wn * 32 + u * 8 + fk * 2 + h;
        if (gj >= N) continue;
        double* c = C + gi * ldc + gj;
        *c = beta == 0.0 ? alpha * acc[t][u][h] : alpha * acc[t][u][h] + beta * *c;
      }
  }
}

static bool pipe_ok(const void* A, int64_t lda, int64_t sA, const void* B, int64_t ldb, int64_t sB) {
  return ((uintptr_t)A % 16) == 0 && ((uintptr_t)B % 16) == 0 && lda % 2 == 0 && ldb % 2 == 0 && sA % 2 == 0 &&
         sB % 2 == 0;
}

template <typename TA, typename TB, bool AT, bool BT>
static void gemm(int64_t M, int64_t N, int64_t K, double alpha, const TA* A, int64_t lda,
                 const TB* B, int64_t ldb, double beta, double* C, int64_t ldc, bool lower,
                 cudaStream_t st, int batch = 1, int64_t sA = 0, int64_t sB = 0, int64_t sC = 0, int kmode = 0) {
  if (M <= 0 || N <= 0) return;
  if constexpr (std::is_same<TA, double>::value && std::is_same<TB, double>::value) {
    static const bool simt = [] {
      const char* e = getenv("GF_DGEMM_SIMT");
      return e && e[0] == '1';
    }();
    // fp64 tensor cores (DMMA) for long reductions; short-K updates (the
    // 128-deep Cholesky trailing updates) are faster on the SIMT tile, whose
    // smaller CTAs fill the machine better (measured at q = 5000 and 20000;
    // at q = 20000 DMMA for the updates: 160 -> 245 ms)
    static const int pipe_mink = [] {   // GF_DGEMM_PIPE_MINK: K from which the pipelined kernel runs (0: never)
      const char* e = getenv("GF_DGEMM_PIPE_MINK");
      return e ? atoi(e) : 512;
    }();
    if (!simt && pipe_mink > 0 && K >= pipe_mink && pipe_ok(A, lda, sA, B, ldb, sB)) {
      static bool attr = false;
      if (!attr) {
        GF_CUDA(cudaFuncSetAttribute(dgemm_pipe_kernel<AT, BT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kPipeSmem));
        attr = true;
      }
      dim3 grid((unsigned)ceil_div(N, PBM), (unsigned)ceil_div(M, PBM), (unsigned)batch);
      dgemm_pipe_kernel<AT, BT><<<grid, 256, kPipeSmem, st>>>(M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, C,
                                                              ldc, sC, lower ? 1 : 0, kmode);
      GF_CHECK_LAUNCH();
      return;
    }
    if (!simt && K >= 512) {
      dim3 grid((unsigned)ceil_div(N, TBN), (unsigned)ceil_div(M, TBM), (unsigned)batch);
      dgemm_tc_kernel<AT, BT><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, C, ldc, sC,
                                                    lower ? 1 : 0, kmode);
      GF_CHECK_LAUNCH();
      return;
    }
  }
  dim3 grid((unsigned)ceil_div(N, GB), (unsigned)ceil_div(M, GB), (unsigned)batch);
  gemm_kernel<TA, TB, AT, BT><<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, sA, B, ldb, sB,
                                                    beta, C, ldc, sC, lower ? 1 : 0);
  GF_CHECK_LAUNCH();
}

// ---------------------------------------------------------- Gram matrix ----
// G = A'A + I (tall) or AA' + I (wide), fp64, lower triangle then mirrored.
__global__ void add_identity_mirror(double* G, int64_t q, int64_t ld) {
  const int64_t i = blockIdx.y * (int64_t)blockDim.y + threadIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= q || j >= q) return;
  if (i == j) G[i * ld + j] += 1.0;
  else if (j > i) G[i * ld + j] = G[j * ld + i];
}

__global__ void mirror_lower(double* G, int64_t q, int64_t ld) {
  const int64_t i = blockIdx.y * (int64_t)blockDim.y + threadIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= q || j >= q || j <= i) return;
  G[i * ld + j] = G[j * ld + i];
}

static dim3 grid2(int64_t q) { return dim3((unsigned)ceil_div(q, 32), (unsigned)ceil_div(q, 8)); }

void gram_accumulate(const gf_matrix* A, bool tall, double* G, int64_t ldg, cudaStream_t st, void* scratch,
                     size_t scratch_bytes, const unsigned* amax_known) {
  const int64_t q = tall ? A->n : A->m;
  if (A->dtype == GF_F32) {
    const float* a = (const float*)A->data;
    const char* env = getenv("GF_GRAM_SIMT");
    if (tall && !(env && env[0] == '1')) {   // tensor cores: tcgen05 split (gf_syrk_tc.cu)
      gram_tf32x3(A, G, ldg, st, scratch, scratch_bytes, amax_known);
      return;
    }
    if (tall) gemm<float, float, true, false>(q, q, A->m, 1.0, a, A->ld, a, A->ld, 0.0, G, ldg, true, st);
    else gemm<float, float, false, true>(q, q, A->n, 1.0, a, A->ld, a, A->ld, 0.0, G, ldg, true, st);
  } else {
    const double* a = (const double*)A->data;
    if (tall && gram_f64_i8(A, G, ldg, st, scratch, scratch_bytes)) return;   // int8 tensor cores
    if (tall) gemm<double, double, true, false>(q, q, A->m, 1.0, a, A->ld, a, A->ld, 0.0, G, ldg, true, st);
    else gemm<double, double, false, true>(q, q, A->n, 1.0, a, A->ld, a, A->ld, 0.0, G, ldg, true, st);
  }
}

void gram_finish(double* G, int64_t q, int64_t ldg, cudaStream_t st) {
  add_identity_mirror<<<grid2(q), dim3(32, 8), 0, st>>>(G, q, ldg);
  GF_CHECK_LAUNCH();
}

// ---------------------------------------------------- blocked Cholesky ----
constexpr int NB = 64;

// Blocked right-looking Cholesky with 128-wide blocks (40 steps at q = 5000):
//   potrf_block  one CTA factors the diagonal block in shared memory, itself
//                right-looking over 16-column micro-panels (warp-level 16x16
//                factor, per-row forward substitution, 4x4 register-blocked
//                trailing update);
//   trsm_rows    one warp per panel row below it, X <- X L_kk^-T, the row in
//                registers (4 columns per lane), L_kk in shared memory;
//   gemm         trailing update G22 -= L21 L21' (lower tiles only).
constexpr int CB = 128, CMB = 16, CSL = CB + 1;
constexpr size_t kCholSmem = (size_t)CB * CSL * sizeof(double);

// 16 x 16 leaf of the diagonal-block factorisation, lane i holding row i in
// registers; pivot J then the rank-1 update of the later columns.  Template
// recursion keeps every register index static (a loop here was left rolled
// by the compiler and put the row in local memory).  One reciprocal square
// root per pivot: the pivots are a serial chain, this is its latency.
template <int J, int K>
__device__ __forceinline__ void leaf_update(double (&r)[CMB], int lane) {
  if constexpr (K < CMB) {
    const double lkj = __shfl_sync(0xffffffffu, r[J], K);
    if (lane >= K) r[K] = fma(-r[J], lkj, r[K]);
    leaf_update<J, K + 1>(r, lane);
  }
}

template <int J>
__device__ __forceinline__ void leaf_pivot(double (&r)[CMB], int lane, double* rinv, int* info, int64_t base) {
  if constexpr (J < CMB) {
    double dj = __shfl_sync(0xffffffffu, r[J], J);
    double ri;
    if (!(dj > 0.0) || !isfinite(dj)) {
      if (lane == 0 && *info == 0) *info = (int)(base + J + 1);
      dj = 1.0;
      ri = 1.0;
    } else {
      ri = rsqrt(dj);
      dj = dj * ri;
    }
    if (lane == J) r[J] = dj;
    if (lane > J) r[J] *= ri;
    if (lane == 0) rinv[J] = ri;
    leaf_update<J, J + 1>(r, lane);
    leaf_pivot<J + 1>(r, lane, rinv, info, base);
  }
}

__global__ void __launch_bounds__(512) potrf_block(double* G, int64_t ld, int64_t k0, int nb, int* info) {
  extern __shared__ double S[];
  __shared__ double rinv[CB];   // reciprocals of the finished pivots (no divisions in the chains)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    const int i = idx / nb, j = idx % nb;
    if (j <= i) S[i * CSL + j] = G[(k0 + i) * ld + k0 + j];
  }
  __syncthreads();
  for (int p = 0; p < nb; p += CMB) {
    const int w = min(CMB, nb - p);
    if (w == CMB) {
      if (warp == 0) {   // full 16 x 16 leaf in registers: lane i holds row p + i
        double r[CMB];
#pragma unroll
        for (int k = 0; k < CMB; ++k) r[k] = (lane < CMB && k <= lane) ? S[(p + lane) * CSL + p + k] : 0.0;
        leaf_pivot<0>(r, lane, rinv + p, info, k0 + p);
        if (lane < CMB)
#pragma unroll
          for (int k = 0; k < CMB; ++k)
            if (k <= lane) S[(p + lane) * CSL + p + k] = r[k];
      }
      __syncthreads();
      const int rows = nb - p - CMB;
      for (int rr = tid; rr < rows; rr += blockDim.x) {   // X <- X L_pp^-T, row in registers
        double* xs = S + (p + CMB + rr) * CSL + p;
        double x[CMB];
#pragma unroll
        for (int c = 0; c < CMB; ++c) x[c] = xs[c];
#pragma unroll
        for (int c = 0; c < CMB; ++c) {
          double sacc = x[c];
#pragma unroll
          for (int t = 0; t < c; ++t) sacc = fma(-x[t], S[(p + c) * CSL + p + t], sacc);
          x[c] = sacc * rinv[p + c];
        }
#pragma unroll
        for (int c = 0; c < CMB; ++c) xs[c] = x[c];
      }
      __syncthreads();
    } else {
    if (warp == 0) {   // w x w diagonal piece, lane i <-> row p + i
      for (int j = 0; j < w; ++j) {
        double* dj = &S[(p + j) * CSL + p + j];
        if (lane == 0) {
          const double v = *dj;
          if (!(v > 0.0) || !isfinite(v)) {
            if (*info == 0) *info = (int)(k0 + p + j + 1);
            *dj = 1.0;
          } else {
            *dj = sqrt(v);
          }
          rinv[p + j] = 1.0 / *dj;
        }
        __syncwarp();
        const double ri = rinv[p + j];
        if (lane > j && lane < w) S[(p + lane) * CSL + p + j] *= ri;
        __syncwarp();
        if (lane > j && lane < w) {
          const double lij = S[(p + lane) * CSL + p + j];
          for (int k = j + 1; k <= lane; ++k) S[(p + lane) * CSL + p + k] -= lij * S[(p + k) * CSL + p + j];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    const int rows = nb - p - w;
    for (int rr = tid; rr < rows; rr += blockDim.x) {   // X <- X L_pp^-T
      double* x = S + (p + w + rr) * CSL + p;
      for (int c = 0; c < w; ++c) {
        double sacc = x[c];
        for (int t = 0; t < c; ++t) sacc -= x[t] * S[(p + c) * CSL + p + t];
        x[c] = sacc * rinv[p + c];
      }
    }
    __syncthreads();
    }
    const int rows = nb - p - w;
    const int nt = (rows + 3) / 4;   // trailing lower update, 4x4 tiles
    const int ntiles = nt * (nt + 1) / 2;
    for (int ti = tid; ti < ntiles; ti += blockDim.x) {
      int bi = (int)((sqrtf(8.f * ti + 1.f) - 1.f) * 0.5f);
      while ((bi + 1) * (bi + 2) / 2 <= ti) ++bi;
      while (bi * (bi + 1) / 2 > ti) --bi;
      const int bj = ti - bi * (bi + 1) / 2;
      const int i0 = p + w + 4 * bi, j0 = p + w + 4 * bj;
      double acc[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
      for (int t = 0; t < w; ++t) {
        double a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a[u] = i0 + u < nb ? S[(i0 + u) * CSL + p + t] : 0.0;
          b[u] = j0 + u < nb ? S[(j0 + u) * CSL + p + t] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (i0 + u < nb && j0 + v <= i0 + u) S[(i0 + u) * CSL + j0 + v] -= acc[u][v];
    }
    __syncthreads();
  }
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    const int i = idx / nb, j = idx % nb;
    G[(k0 + i) * ld + k0 + j] = j <= i ? S[i * CSL + j] : 0.0;
  }
}

// Panel rows r >= k0 + nb: x <- x L_kk^-T, one warp per row; lane l holds
// columns l, l + 32, l + 64, l + 96 of x.  Column c is finished by the lane
// owning it, broadcast, and subtracted from the later columns (right-looking).
__global__ void __launch_bounds__(512) trsm_rows(double* G, int64_t ld, int64_t q, int64_t k0, int nb) {
  extern __shared__ double Ls[];
  __shared__ double rinv[CB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    const int i = idx / nb, j = idx % nb;
    if (j <= i) Ls[i * CSL + j] = G[(k0 + i) * ld + k0 + j];
  }
  for (int c = tid; c < nb; c += blockDim.x) rinv[c] = 1.0 / G[(k0 + c) * ld + k0 + c];
  __syncthreads();
  const int nw = blockDim.x >> 5;
  for (int64_t r = k0 + nb + (int64_t)blockIdx.x * nw + warp; r < q; r += (int64_t)gridDim.x * nw) {
    double* row = G + r * ld + k0;
    double x[CB / 32];
#pragma unroll
    for (int i = 0; i < CB / 32; ++i) x[i] = lane + 32 * i < nb ? row[lane + 32 * i] : 0.0;
#pragma unroll
    for (int sl = 0; sl < CB / 32; ++sl) {
      for (int o = 0; o < 32; ++o) {
        const int c = 32 * sl + o;
        if (c >= nb) break;
        double xc = __shfl_sync(0xffffffffu, x[sl], o);
        xc *= rinv[c];
        if (lane == o) x[sl] = xc;
#pragma unroll
        for (int i = 0; i < CB / 32; ++i) {
          const int t = lane + 32 * i;
          if (t > c && t < nb) x[i] -= xc * Ls[t * CSL + c];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CB / 32; ++i)
      if (lane + 32 * i < nb) row[lane + 32 * i] = x[i];
  }
}

__global__ void zero_upper(double* G, int64_t q, int64_t ld) {
  const int64_t i = blockIdx.y * (int64_t)blockDim.y + threadIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < q && j < q && j > i) G[i * ld + j] = 0.0;
}

// In-place lower Cholesky of G (fp64, q x q, row stride ld); upper part zeroed.
// Returns 0 or the 1-based index of the first non-positive pivot.
int cholesky(double* G, int64_t q, int64_t ld, int* d_info, cudaStream_t st) {
  GF_CUDA(cudaFuncSetAttribute(potrf_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCholSmem));
  GF_CUDA(cudaFuncSetAttribute(trsm_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCholSmem));
  int sms = 148;
  {
    int dev = 0;
    GF_CUDA(cudaGetDevice(&dev));
    GF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  GF_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int), st));
  const char* vb = getenv("GF_VERBOSE_CHOL");   // potrf / trsm / update split (one stream)
  const bool prof = vb && vb[0] == '1';
  std::vector<cudaEvent_t> ev;
  auto mark = [&]() {
    if (!prof) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.push_back(e);
  };
  mark();
  // Depth-1 lookahead: the trailing update of step s is split into (a) the
  // next panel's columns, on the caller's stream, and (b) the columns after
  // it, on a second stream -- so potrf(s+1) and trsm(s+1), the serial chain
  // of small kernels, run while (b)(s) updates the bulk of the trailing
  // matrix.  (a)(s) waits for (b)(s-1), the other writer of panel s+1's
  // columns; potrf(s+1) follows (a)(s) in stream order.  (The verbose phase
  // split keeps one stream.)
  // The chain (potrf, trsm, next panel) runs on a high-priority stream so its
  // small grids are scheduled ahead of the bulk update's remaining CTAs.
  static std::mutex aux_mu;
  static cudaStream_t aux_by_dev[64] = {}, crit_by_dev[64] = {};
  cudaStream_t aux = nullptr, crit = nullptr;
  {
    int dev = 0;
    GF_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(aux_mu);
    if (aux_by_dev[dev & 63] == nullptr) {
      int lo = 0, hi = 0;
      GF_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      GF_CUDA(cudaStreamCreateWithPriority(&aux_by_dev[dev & 63], cudaStreamNonBlocking, lo));
      GF_CUDA(cudaStreamCreateWithPriority(&crit_by_dev[dev & 63], cudaStreamNonBlocking, hi));
    }
    aux = aux_by_dev[dev & 63];
    crit = crit_by_dev[dev & 63];
  }
  cudaEvent_t ev_t = nullptr, ev_b = nullptr;
  const bool look = !prof;
  cudaStream_t caller = st;
  if (look) {
    GF_CUDA(cudaEventCreateWithFlags(&ev_t, cudaEventDisableTiming));
    GF_CUDA(cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming));
    GF_CUDA(cudaEventRecord(ev_t, caller));   // G and d_info are ready
    GF_CUDA(cudaStreamWaitEvent(crit, ev_t, 0));
    st = crit;
  }
  bool b_pending = false;
  // Two-level blocking (GF_CHOL_SP; default 512 from q = 8192, else one level): columns go
  // in super-panels of SP.  Inside one, each 128-column step updates only the
  // super-panel's later columns (every row below: the next steps' TRSM needs
  // them); the trailing matrix past the super-panel takes all SP columns'
  // contributions in one K = SP product, long enough for the pipelined DMMA
  // GEMM (30 TF/s at K = 512 against ~16 for the 128-deep SIMT updates).
  // The lookahead is the one-level scheme's at super-panel granularity: (a)
  // the next super-panel's columns on the chain stream, (b) the rest on aux.
  // Measured (C3, q = 20000): one level 175-205 ms, SP = 512 164 ms, 256 and
  // 1024 slower (529 / 377 ms: K below the pipelined kernel's range, resp.
  // a longer serial chain); at q = 5000 one level is faster (7.0 vs 7.4 ms).
  static const int64_t sp_env = [] {
    const char* e = getenv("GF_CHOL_SP");
    return e ? (int64_t)atoll(e) : (int64_t)-1;
  }();
  const int64_t sp_req = sp_env >= 0 ? sp_env : (q >= 8192 ? 512 : 0);
  const int64_t SP = sp_req >= 2 * CB && sp_req % CB == 0 ? sp_req : 0;
  if (SP > 0 && q > SP) {
    for (int64_t K0 = 0; K0 < q; K0 += SP) {
      const int64_t pe = std::min<int64_t>(K0 + SP, q);
      for (int64_t k0 = K0; k0 < pe; k0 += CB) {
        const int nb = (int)std::min<int64_t>(CB, q - k0);
        potrf_block<<<1, 512, kCholSmem, st>>>(G, ld, k0, nb, d_info);
        GF_CHECK_LAUNCH();
        mark();
        const int64_t rest = q - k0 - nb;
        if (rest <= 0) break;
        const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(rest, 16), sms);
        trsm_rows<<<grid, 512, kCholSmem, st>>>(G, ld, q, k0, nb);
        GF_CHECK_LAUNCH();
        mark();
        const int64_t wc = pe - (k0 + nb);   // the super-panel's later columns
        if (wc > 0) {
          double* L21 = G + (k0 + nb) * ld + k0;
          gemm<double, double, false, true>(rest, wc, nb, -1.0, L21, ld, L21, ld, 1.0, G + (k0 + nb) * ld + k0 + nb,
                                            ld, true, st);
          mark();
        }
      }
      const int64_t rest = q - pe;
      if (rest <= 0) break;
      const int64_t kw = pe - K0;
      const double* L21 = G + pe * ld + K0;
      double* G22 = G + pe * ld + pe;
      if (!look) {
        gemm<double, double, false, true>(rest, rest, kw, -1.0, L21, ld, L21, ld, 1.0, G22, ld, true, st);
        mark();
        continue;
      }
      const int64_t na = std::min<int64_t>(SP, rest);
      const int64_t rb = rest - na;
      if (rb > 0) {
        GF_CUDA(cudaEventRecord(ev_t, st));
        GF_CUDA(cudaStreamWaitEvent(aux, ev_t, 0));
      }
      if (b_pending) GF_CUDA(cudaStreamWaitEvent(st, ev_b, 0));
      gemm<double, double, false, true>(rest, na, kw, -1.0, L21, ld, L21, ld, 1.0, G22, ld, true, st);
      b_pending = false;
      if (rb > 0) {
        const double* L21b = L21 + na * ld;
        gemm<double, double, false, true>(rb, rb, kw, -1.0, L21b, ld, L21b, ld, 1.0, G22 + na * ld + na, ld, true,
                                          aux);
        GF_CUDA(cudaEventRecord(ev_b, aux));
        b_pending = true;
      }
    }
  } else
  for (int64_t k0 = 0; k0 < q; k0 += CB) {
    const int nb = (int)std::min<int64_t>(CB, q - k0);
    potrf_block<<<1, 512, kCholSmem, st>>>(G, ld, k0, nb, d_info);
    GF_CHECK_LAUNCH();
    mark();
    const int64_t rest = q - k0 - nb;
    if (rest <= 0) break;
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(rest, 16), sms);
    trsm_rows<<<grid, 512, kCholSmem, st>>>(G, ld, q, k0, nb);
    GF_CHECK_LAUNCH();
    mark();
    double* L21 = G + (k0 + nb) * ld + k0;
    double* G22 = G + (k0 + nb) * ld + k0 + nb;
    if (!look) {
      gemm<double, double, false, true>(rest, rest, nb, -1.0, L21, ld, L21, ld, 1.0, G22, ld, true, st);
      mark();
      continue;
    }
    const int64_t na = std::min<int64_t>(CB, rest);   // (a): the next panel's columns, every row below
    const int64_t rb = rest - na;                       // (b): the columns after it
    if (rb > 0) {
      GF_CUDA(cudaEventRecord(ev_t, st));               // L21 of this step is final
      GF_CUDA(cudaStreamWaitEvent(aux, ev_t, 0));
    }
    if (b_pending) GF_CUDA(cudaStreamWaitEvent(st, ev_b, 0));   // (b) of the previous step
    gemm<double, double, false, true>(rest, na, nb, -1.0, L21, ld, L21, ld, 1.0, G22, ld, true, st);
    b_pending = false;
    if (rb > 0) {
      const double* L21b = L21 + na * ld;
      gemm<double, double, false, true>(rb, rb, nb, -1.0, L21b, ld, L21b, ld, 1.0, G22 + na * ld + na, ld, true, aux);
      GF_CUDA(cudaEventRecord(ev_b, aux));
      b_pending = true;
    }
  }
  if (look && b_pending) GF_CUDA(cudaStreamWaitEvent(st, ev_b, 0));
  if (look) {   // back on the caller's stream
    GF_CUDA(cudaEventRecord(ev_t, crit));
    GF_CUDA(cudaStreamWaitEvent(caller, ev_t, 0));
    st = caller;
  }
  zero_upper<<<grid2(q), dim3(32, 8), 0, st>>>(G, q, ld);
  GF_CHECK_LAUNCH();
  int info = 0;
  GF_CUDA(cudaMemcpyAsync(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  if (ev_t) cudaEventDestroy(ev_t);
  if (ev_b) cudaEventDestroy(ev_b);
  return info;
}

// ----------------------------------------------- triangular inverse W=L^-1 --
// Level 0: invert every diagonal NB-block in place (one CTA per block,
// thread c solves L w = e_c with w in a thread-local array).
__global__ void trtri_diag(double* L, int64_t ld, int64_t q) {
  __shared__ double S[NB][NB + 1];
  const int64_t k0 = (int64_t)blockIdx.x * NB;
  const int nb = (int)min((int64_t)NB, q - k0);
  const int tid = threadIdx.x;
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    const int i = idx / nb, j = idx % nb;
    S[i][j] = L[(k0 + i) * ld + k0 + j];
  }
  __syncthreads();
  if (tid < nb) {
    const int c = tid;
    double w[NB];
    for (int r = 0; r < nb; ++r) {
      if (r < c) { w[r] = 0.0; continue; }
      double s = (r == c) ? 1.0 : 0.0;
      for (int t = c; t < r; ++t) s -= S[r][t] * w[t];
      w[r] = s / S[r][r];
    }
    for (int r = 0; r < nb; ++r) L[(k0 + r) * ld + k0 + c] = w[r];
  }
}

// In place: L (lower, fp64) -> W = L^-1.  tmp: q x ld scratch.
void trtri(double* L, int64_t q, int64_t ld, double* tmp, cudaStream_t st) {
  trtri_diag<<<(unsigned)ceil_div(q, NB), NB, 0, st>>>(L, ld, q);
  GF_CHECK_LAUNCH();
  for (int64_t s = NB; s < q; s *= 2) {
    const int64_t pair = 2 * s;
    const int64_t full = q / pair;  // pairs with both halves of size s
    // batched over full pairs: T = L21 W11; W21 = -W22 T
    if (full > 0) {
      const double* L21 = L + s * ld;          // rows [s, 2s), cols [0, s) of pair 0
      const double* W11 = L;                   // rows [0, s), cols [0, s)
      double* T = tmp;
      gemm<double, double, false, false>(s, s, s, 1.0, L21, ld, W11, ld, 0.0, T, ld, false, st,
                                         (int)full, pair * ld + pair, pair * ld + pair, pair * ld + pair, 1);
      const double* W22 = L + s * ld + s;
      double* W21 = L + s * ld;
      gemm<double, double, false, false>(s, s, s, -1.0, W22, ld, T, ld, 0.0, W21, ld, false, st,
                                         (int)full, pair * ld + pair, pair * ld + pair, pair * ld + pair, 2);
    }
    // ragged last pair: first half size s, second half size r2 < s
    const int64_t p0 = full * pair;
    const int64_t r2 = q - p0 - s;
    if (r2 > 0) {
      const double* L21 = L + (p0 + s) * ld + p0;
      const double* W11 = L + p0 * ld + p0;
      double* T = tmp + p0 * ld + p0;
      gemm<double, double, false, false>(r2, s, s, 1.0, L21, ld, W11, ld, 0.0, T, ld, false, st, 1, 0, 0, 0, 1);
      const double* W22 = L + (p0 + s) * ld + p0 + s;
      double* W21 = L + (p0 + s) * ld + p0;
      gemm<double, double, false, false>(r2, s, r2, -1.0, W22, ld, T, ld, 0.0, W21, ld, false, st, 1, 0, 0, 0, 2);
    }
  }
}

// G^-1 = W' W from W = L^-1 (lower); lower triangle computed, then mirrored.
void inverse_from_factor_inv(const double* W, int64_t q, int64_t ld, double* Ginv, cudaStream_t st) {
  gemm<double, double, true, false>(q, q, q, 1.0, W, ld, W, ld, 0.0, Ginv, ld, true, st, 1, 0, 0, 0, 3);
  mirror_lower<<<grid2(q), dim3(32, 8), 0, st>>>(Ginv, q, ld);
  GF_CHECK_LAUNCH();
}

template <typename T>
__global__ void convert_pad(const double* __restrict__ src, int64_t lds, T* __restrict__ dst,
                            int64_t ldd, int64_t rows, int64_t cols) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y)
    for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < ldd; j += (int64_t)gridDim.x * blockDim.x)
      dst[i * ldd + j] = j < cols ? (T)src[i * lds + j] : (T)0;
}

void store_matrix(const double* src, int64_t lds, int dtype, void* dst, int64_t ldd, int64_t rows,
                  int64_t cols, cudaStream_t st) {
  if (rows <= 0) return;
  dim3 grid((unsigned)std::min<int64_t>(ceil_div(ldd, 256), 64), (unsigned)std::min<int64_t>(rows, 65535));
  if (dtype == GF_F32) convert_pad<float><<<grid, 256, 0, st>>>(src, lds, (float*)dst, ldd, rows, cols);
  else convert_pad<double><<<grid, 256, 0, st>>>(src, lds, (double*)dst, ldd, rows, cols);
  GF_CHECK_LAUNCH();
}

}  // namespace gf
