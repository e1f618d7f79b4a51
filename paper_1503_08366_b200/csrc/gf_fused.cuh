// Fused single-pass ADMM row/column kernel (tall problems, rows that fit in
// shared memory).
//
// The reference reads A four times per iteration (two projection matvecs plus
// the two residual matvecs on a second, unscaled copy; solver.py:197-198,
// projection.py:121-122), and the plain restatement still needs two passes:
// y+ = A_hat x+ (row pass) and A_hat' [c_y, nu^] (column pass).  But c_y and
// nu^ of row i depend only on row i's own dot products, so the column pass can
// consume each row once its epilogue is done -- while the row is still on
// chip.  One iteration then streams A_hat from HBM exactly once.
//
// Structure: one persistent CTA per SM over a contiguous row range; a ring of
// NSLOT row slots in shared memory filled by TMA bulk copies (cp.async.bulk,
// L2 evict_first, one mbarrier per slot) issued by a producer warp.  CW
// compute warps (plan_fused: the fewest that keep <= 5 16-byte vectors per
// thread, 8 at n = 5000) own fixed column vectors (x^, x^_1/2 and the column
// accumulators live in registers for the whole kernel; fp32 rows use packed
// FFMA2); three epilogue warps run the fp64 y side.  Rows move in groups of
// TR through a three-stage software pipeline whose hand-offs are all
// mbarriers (no CTA-wide barrier after setup):
//
//   compute warps   R(t)   dots of group t                    -> red_s[t % 3]
//                   C(t-2) A' [c_y, nu^] of group t-2 with w_s[(t-2) % 3],
//                          then release its slots to the producer
//   epilogue warps  E(t)   (warp CW + t % 3) reduce red_s[t % 3]; y side of
//                          group t (Epi::mid -> w_s, then Epi::tail)
//   producer warp          refill released slots with the rows NSLOT ahead
//
// so the serial per-row epilogue (fp64 prox, divisions, global stores) runs
// concurrently with the row and column passes of other groups.  Three groups
// are resident; NSLOT - 3*TR rows are in flight from HBM.  The first ring fill
// is issued before the programmatic-dependency wait (A_hat is constant).
#pragma once

#include <algorithm>

#include "gf_common.cuh"
#include "gf_gemv.cuh"

namespace gf {

constexpr int kMaxSlots = 32;
// static shared memory of the kernels (barriers, hand-off buffers, the Z
// tail's reduction scratch) comes out of the same per-block limit as the ring
constexpr size_t kStaticSmemReserve = 16384;
// Epilogue warps: warp e takes the groups ge = e (mod kFusedEpi) and owns
// hand-off buffer e, so each warp has kFusedEpi row-pass periods per group
// while the latency from R(ge) to its weights stays under the two-period lag.
// Three: 16 + 3 + 1 = 20 warps keeps 5 warps per SM sub-partition (96 registers
// per thread); with 20 compute warps the CTA has 24 warps (80 registers).
#ifndef GF_FUSED_NE
#define GF_FUSED_NE 3
#endif
constexpr int kFusedEpiMax = 8;
__host__ __device__ constexpr int fused_epi(int cw) { return GF_FUSED_NE; }
// CTA size for CW compute warps: + the epilogue warps + 1 producer warp
__host__ __device__ constexpr int fused_threads(int cw) { return (cw + fused_epi(cw) + 1) * 32; }
// The lagged cluster pass (below) runs more epilogue warps.
constexpr int kLagEpi = 7;
__host__ __device__ constexpr int fused_epi_lag(int cw, int lag) { return lag > 0 ? kLagEpi : fused_epi(cw); }
__host__ __device__ constexpr int fused_threads_lag(int cw, int lag) { return (cw + fused_epi_lag(cw, lag) + 1) * 32; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// Waiting threads are suspended (up to this many ns, woken early when the
// phase completes) instead of spinning, so blocked warps do not take issue
// slots from the ones doing work on the same sub-partition.
#ifndef GF_SUSPEND_NS
#define GF_SUSPEND_NS 20000
#endif
constexpr unsigned kSuspendNs = GF_SUSPEND_NS;

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(kSuspendNs)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// The same on precomputed 32-bit shared addresses (no generic->shared
// conversion per call in the hot loops).
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity), "r"(kSuspendNs)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t addr, float4*) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ double2 lds128(uint32_t addr, double2*) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// TMA bulk copy global -> shared, completion counted on `bar` (tx bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// The same without a cache-policy hint (normal L2 priority).
__device__ __forceinline__ void bulk_g2s_nohint(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ float vdot(const float4& a, const float4& b, float s) {
  s = fmaf(a.x, b.x, s);
  s = fmaf(a.y, b.y, s);
  s = fmaf(a.z, b.z, s);
  return fmaf(a.w, b.w, s);
}
__device__ __forceinline__ double vdot(const double2& a, const double2& b, double s) {
  s = fma(a.x, b.x, s);
  return fma(a.y, b.y, s);
}
// fp32 rows use Blackwell's packed FFMA2 (fma.rn.f32x2): half the FMA
// instructions of the scalar form for both passes.
__device__ __forceinline__ void vaxpy(float4& acc, const float4& a, float w) {
  const float2 ww = make_float2(w, w);
  const float2 lo = __ffma2_rn(make_float2(a.x, a.y), ww, make_float2(acc.x, acc.y));
  const float2 hi = __ffma2_rn(make_float2(a.z, a.w), ww, make_float2(acc.z, acc.w));
  acc = make_float4(lo.x, lo.y, hi.x, hi.y);
}
// Row-pass dot accumulators: a float2 pair (even / odd lanes of the vector)
// for fp32, a scalar for fp64.
template <typename T> struct DotAcc;
template <> struct DotAcc<float> { using type = float2; };
template <> struct DotAcc<double> { using type = double; };
__device__ __forceinline__ float2 dot_acc(const float4& a, const float4& b) {
  const float2 s = __fmul2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
  return __ffma2_rn(make_float2(a.z, a.w), make_float2(b.z, b.w), s);
}
__device__ __forceinline__ double dot_acc(const double2& a, const double2& b) { return fma(a.y, b.y, a.x * b.x); }
__device__ __forceinline__ float2 dot_add(float2 s, float2 t) { return make_float2(s.x + t.x, s.y + t.y); }
__device__ __forceinline__ double dot_add(double s, double t) { return s + t; }
__device__ __forceinline__ float dot_fin(float2 s) { return s.x + s.y; }
__device__ __forceinline__ double dot_fin(double s) { return s; }
__device__ __forceinline__ void vaxpy(double2& acc, const double2& a, double w) {
  acc.x = fma(a.x, w, acc.x);
  acc.y = fma(a.y, w, acc.y);
}

struct FusedPlan {
  int cw = 0;        // compute warps (template instance: 8, 12, 16 or 20)
  int ne = 0;        // epilogue warps (= partial records per CTA)
  int nv = 0;        // 16-byte vectors per thread per row (template instance)
  int nslot = 0;     // rows resident in shared memory
  int tr = 0;        // rows per group (template instance: 1, 2 or 4)
  int grid = 0;      // CTAs (one per SM)
  size_t smem = 0;   // dynamic shared memory bytes
  bool ok = false;
};

inline FusedPlan plan_fused(int64_t m, int64_t ld, int esize, int sms, size_t smem_max, int max_slots = kMaxSlots) {
  FusedPlan p;
  const int vn = 16 / esize;
  const int64_t nvec = ld / vn;
  // The fewest compute warps that keep the vectors per thread at <= 5
  // (measured on B200, tools/fused_bench.cu: fewer, wider warps leave issue
  // slots to the fp64 epilogue warps and cut the per-row sync overhead;
  // 8 warps x 5 vectors beats 20 x 2 by 15 % on the 200000 x 5000 fp32 row).
  // (16 and 20 compute warps: at most 4 vectors, the register budget of the
  // larger CTA; beyond 20 x 4 the 5- and 6-vector instances spill a little)
  p.cw = 20;
  for (int cw : {8, 12, 16, 20})
    if (ceil_div(nvec, cw * 32) <= (cw <= 12 ? 5 : 4)) { p.cw = cw; break; }
  p.nv = (int)ceil_div(nvec, p.cw * 32);
  p.ne = fused_epi(p.cw);
  const size_t row_bytes = (size_t)ld * esize;
  const size_t budget = smem_max > kStaticSmemReserve ? smem_max - kStaticSmemReserve : 0;
  p.nslot = (int)std::min<size_t>(std::min(max_slots, kMaxSlots), budget / row_bytes);
  // keep >= 2 rows and >= 48 KB of TMA prefetch beyond the three resident groups
  const int want_pf = std::max<int>(2, (int)ceil_div(48 * 1024, (int64_t)row_bytes));
  p.tr = 0;
  for (int tr : {4, 2, 1})
    if (3 * tr + want_pf <= p.nslot || (tr == 1 && 3 + 1 <= p.nslot)) { p.tr = tr; break; }
  p.grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, m));
  p.smem = (size_t)p.nslot * row_bytes;
  p.ok = p.nv >= 1 && p.nv <= 6 && p.tr >= 1 && m > 0;
  return p;
}

// All-lane sum of K values per lane in 5 + (K-1) shuffles instead of 5K: the
// first log2(K) butterfly stages split the values between lane halves, so
// after them lane l holds the partial of value (l >> (5 - log2 K))
// ... of its half; the remaining stages are plain xor reductions.  Returns, in
// lanes whose index selects value q, the full sum of value q; the caller reads
// value q from lane q << (5 - log2 K).
template <int K, typename T>
__device__ __forceinline__ T warp_multi_sum(T (&v)[K], int lane) {
  static_assert(K == 1 || K == 2 || K == 4 || K == 8, "K must be 1, 2, 4 or 8");
  constexpr int LG = K == 1 ? 0 : (K == 2 ? 1 : (K == 4 ? 2 : 3));
#pragma unroll
  for (int s = 0; s < LG; ++s) {
    const int off = 16 >> s;                 // 16, 8, 4
    const bool upper = (lane & off) != 0;
    constexpr int dummy = 0;
    (void)dummy;
    const int half = K >> (s + 1);           // values kept after this stage
#pragma unroll
    for (int q = 0; q < half; ++q) {
      // lanes in the lower half keep value q, the upper half keeps value q + half
      const T send = upper ? v[q] : v[q + half];
      const T keep = upper ? v[q + half] : v[q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  T r = v[0];
#pragma unroll
  for (int off = 16 >> LG; off > 0; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
  return r;
}

// Work run by every thread of every CTA after the pass (the solver's Z step,
// ZTail in gf_solver.cu); NoTail: none.
struct NoTail {
  __device__ bool on() const { return false; }
  __device__ void run() const {}
};

// Epi must provide: NR, active(), begin(), RowIn, load_in(i), Mid,
// mid(in, dots, w0, w1) (the column-pass weights: critical path) and
// tail(i, in, dots, mid, red, flags) (stores, reductions)  -- YEpi does.
//
// Warp roles (no CTA-wide barrier after setup; every hand-off is an mbarrier),
// shown for CW = 16 compute warps:
//   warps 0..15  compute   R(t): dots of group t -> red_s[t&1] (arrive redf)
//                          C(t-2): column pass with w_s[t&1]  (wait wf, arrive we;
//                          arrive sfree[slot] per row consumed)
//   warps 16,17  epilogue  warp 16+b takes the groups of parity b (buffers b):
//                          wait redf -> reduce -> arrive rede; wait we ->
//                          y-side epilogue -> w_s -> arrive wf.  Two epilogue
//                          warps double the rows in flight through the serial
//                          fp64 epilogue, which is latency- not throughput-bound.
//   warp 18      producer  wait sfree[slot] -> TMA bulk copy of the row NSLOT ahead
// Dev instrumentation (tools/fused_bench.cu): per-CTA cycle counters of the
// pipeline waits and epilogue phases; compiled out of the library.
#ifdef GF_FUSED_TRACE
__device__ unsigned long long gf_fused_trace[148 * 16];
#define GF_TR_T0() const long long tr_t0_ = clock64()
#define GF_TR_ADD(slot, t0) atomicAdd(&gf_fused_trace[blockIdx.x * 16 + (slot)], (unsigned long long)(clock64() - (t0)))
#else
#define GF_TR_T0() (void)0
#define GF_TR_ADD(slot, t0) (void)0
#endif

template <typename T, int NV, int TR, int CW, class Epi, class Tail = NoTail>
__global__ void __launch_bounds__(fused_threads(CW), 1)
fused_rowcol_kernel(const T* __restrict__ A, int64_t rows, int64_t ld, const T* __restrict__ x0,
                    const T* __restrict__ x1, Epi epi, int nslot, double* __restrict__ rpart,
                    double* __restrict__ cpart, Tail tail = Tail{}) {
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
  constexpr int NR = Epi::NR;
  constexpr int K = 2 * TR;
  constexpr int LGK = K == 2 ? 1 : (K == 4 ? 2 : 3);
  constexpr int kFusedWarps = CW;
  constexpr int kFusedThreads = CW * kWarp;
  constexpr int NE = fused_epi(CW);
  constexpr int kEpiWarp = CW;          // CW .. CW + NE - 1
  constexpr int kProdWarp = CW + NE;
  static_assert(CW <= 32, "one epilogue lane per compute warp");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxSlots], sfree[kMaxSlots];
  __shared__ __align__(8) uint64_t redf[NE], rede[NE], wf[NE], we[NE];
  __shared__ T red_s[NE][kFusedWarps][K];
  __shared__ T w_s[NE][TR][2];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nvec = ld / VN;
  const unsigned rb = (unsigned)(ld * sizeof(T));
  const int64_t r0 = rows * blockIdx.x / gridDim.x;   // contiguous, balanced row range
  const int64_t r1 = rows * (blockIdx.x + 1) / gridDim.x;
  const int nr = (int)(r1 - r0);
  const int ng = (nr + TR - 1) / TR;

  if (tid == 0) {
    for (int s = 0; s < nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sfree[s], kFusedWarps);
    }
    for (int b = 0; b < NE; ++b) {
      mbar_init(&redf[b], kFusedWarps);
      mbar_init(&rede[b], 1);
      mbar_init(&wf[b], 1);
      mbar_init(&we[b], kFusedWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kProdWarp) {
    // ===================== producer warp =====================
    // A_hat does not depend on the previous kernel: the first ring fill is
    // issued before the programmatic-dependency wait (overlapping the
    // predecessor's tail); if the solve has ended meanwhile the copies are
    // drained before the CTA exits.
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int pre = min(nslot, nr);
      for (int j = 0; j < pre; ++j) {
        mbar_arrive_expect_tx(&full[j], rb);
        bulk_g2s(smem_raw + j * rb, A + (r0 + j) * ld, rb, &full[j], pol);
      }
      pdl_wait();
      pdl_trigger();
      if (!epi.active()) {
        for (int j = 0; j < pre; ++j) mbar_wait(&full[j], 0u);
        return;
      }
      int slot = pre == nslot ? 0 : pre;
      for (int j = pre; j < nr; ++j) {
#ifdef GF_FUSED_TRACE
        long long c0 = clock64();
#endif
        if (j >= nslot) mbar_wait(&sfree[slot], (unsigned)(((j / nslot) - 1) & 1));
#ifdef GF_FUSED_TRACE
        GF_TR_ADD(11, c0);
#endif
        mbar_arrive_expect_tx(&full[slot], rb);
        bulk_g2s(smem_raw + slot * rb, A + (r0 + j) * ld, rb, &full[slot], pol);
        if (++slot == nslot) slot = 0;
      }
    }
  } else {
  pdl_wait();
  if (!epi.active()) return;
  if (warp >= kEpiWarp && warp < kEpiWarp + NE) {
    // ===================== epilogue warps =====================
    const int par = warp - kEpiWarp;   // this warp's groups and buffer
    epi.begin();
    double ered[NR > 0 ? NR : 1];
#pragma unroll
    for (int k = 0; k < (NR > 0 ? NR : 1); ++k) ered[k] = 0.0;
    unsigned eflags = 0;
    typename Epi::RowIn in{};
    if (lane < TR && par * TR + lane < nr) in = epi.load_in(r0 + par * TR + lane);
    for (int ge = par; ge < ng; ge += NE) {
      const int b = par;
      const unsigned use = (unsigned)(ge / NE);
#ifdef GF_FUSED_TRACE
      long long c0 = clock64();
#endif
      mbar_wait_u32(smem_u32(&redf[b]), use & 1u);
#ifdef GF_FUSED_TRACE
      long long c1 = clock64();
      if (lane == 0) GF_TR_ADD(0, c0);
#endif
      // fixed-order tree over the CW compute warps: lane w loads warp w's partials
      constexpr int RW = CW <= 16 ? 16 : 32;   // shuffle width covering the warps
      double v[K];
#pragma unroll
      for (int q = 0; q < K; ++q) v[q] = lane < kFusedWarps ? (double)red_s[b][lane][q] : 0.0;
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&rede[b], 0);   // red_s[b] may be rewritten
#pragma unroll
      for (int q = 0; q < K; ++q)
#pragma unroll
        for (int o = RW / 2; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o, RW);
#ifdef GF_FUSED_TRACE
      if (lane == 0) GF_TR_ADD(2, c1);
      c1 = clock64();
#endif
      if (use >= 1) mbar_wait_u32(smem_u32(&we[b]), (use - 1) & 1u);    // w_s[b] consumed by C(ge-NE)
#ifdef GF_FUSED_TRACE
      if (lane == 0) GF_TR_ADD(3, c1);
      c1 = clock64();
#endif
      const int g = min(TR, nr - ge * TR);
      double dots[2] = {0.0, 0.0};
#pragma unroll
      for (int rr = 0; rr < TR; ++rr)
        if (rr == lane) { dots[0] = v[2 * rr]; dots[1] = v[2 * rr + 1]; }
      // critical path first: the column-pass weights, handed off before the
      // row's stores and reductions (Epi::tail) run
      typename Epi::Mid md{};
      if (lane < g) {
        double w0, w1;
        md = epi.mid(in, dots, w0, w1);
        w_s[b][lane][0] = (T)w0;
        w_s[b][lane][1] = (T)w1;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&wf[b], 0);
#ifdef GF_FUSED_TRACE
      if (lane == 0) GF_TR_ADD(4, c1);
      c1 = clock64();
#endif
      if (lane < g) epi.tail(r0 + (int64_t)ge * TR + lane, in, dots, md, ered, eflags);
      const int jn = (ge + NE) * TR + lane;   // prefetch the inputs of this warp's next group
      if (lane < TR && jn < nr) in = epi.load_in(r0 + jn);
#ifdef GF_FUSED_TRACE
      __syncwarp();
      if (lane == 0) GF_TR_ADD(5, c1);
      if (lane == 0) GF_TR_ADD(6, c0);
#endif
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) ered[k] = warp_sum(ered[k]);
    eflags = warp_or(eflags);
    if (lane == 0) {   // one partial record per epilogue warp: rpart[NE * cta + par]
      double* out = rpart + (NE * (int64_t)blockIdx.x + par) * (NR + 1);
      for (int k = 0; k < NR; ++k) out[k] = ered[k];
      out[NR] = (double)eflags;
    }
  } else {

  // ===================== compute warps =====================
  // Thread tid owns the 16-byte column vectors c = tid + v * CW * 32.  Only
  // the last (v = NV - 1) can fall past the row end (NV = ceil(nvec / (CW*32)));
  // its smem index is clamped onto a vector of the same row (finite: A is
  // validated finite) and its x entries are zero, so it adds exact zeros to
  // the dots, and its column accumulators are never stored -- the inner loops
  // carry no bounds branches.  All shared addresses are 32-bit and hoisted.
  V xa[NV], xb[NV], ca[NV], cb[NV];
  uint32_t voff[NV];
  {
    const V* xv0 = reinterpret_cast<const V*>(x0);
    const V* xv1 = reinterpret_cast<const V*>(x1);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = tid + v * kFusedThreads;
      const bool ok = c < (int)nvec;
      voff[v] = (uint32_t)(ok ? c : (int)nvec - 1) * 16u;
      xa[v] = ok ? xv0[c] : V{};
      xb[v] = ok ? xv1[c] : V{};
      ca[v] = V{};
      cb[v] = V{};
    }
  }
  const uint32_t ring0 = smem_u32(smem_raw);
  const uint32_t full0 = smem_u32(full), sfree0 = smem_u32(sfree);
  const uint32_t redf0 = smem_u32(redf), rede0 = smem_u32(rede), wf0 = smem_u32(wf), we0 = smem_u32(we);
  const bool red_writer = (lane & ((32 >> LGK) - 1)) == 0;
  T* const red_dst = &red_s[0][warp][lane >> (5 - LGK)];   // + b * CW * K
  int slotR = 0, slotC = 0;
  unsigned phaseR = 0;
  int jR = 0, jC = 0;
  int bR = 0, bC = 0;            // hand-off buffer of R(t) / C(t-2): t mod NE
  unsigned useR = 0, useC = 0;   // its use count: t / NE
  for (int t = 0; t < ng + 2; ++t) {
    if (t < ng) {   // ---- R(t) ----
      T s[K];
#pragma unroll
      for (int rr = 0; rr < TR; ++rr) {
        s[2 * rr] = 0;
        s[2 * rr + 1] = 0;
        if (jR < nr) {
#ifdef GF_FUSED_TRACE
          long long c0 = clock64();
#endif
          mbar_wait_u32(full0 + 8u * slotR, phaseR);
#ifdef GF_FUSED_TRACE
          if (tid == 0) GF_TR_ADD(8, c0);
#endif
          const uint32_t row = ring0 + (uint32_t)slotR * rb;
          typename DotAcc<T>::type p0[NV], p1[NV];
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const V a = lds128(row + voff[v], (V*)nullptr);
            p0[v] = dot_acc(a, xa[v]);
            p1[v] = dot_acc(a, xb[v]);
          }
#pragma unroll
          for (int v = 1; v < NV; ++v) { p0[0] = dot_add(p0[0], p0[v]); p1[0] = dot_add(p1[0], p1[v]); }
          s[2 * rr] = dot_fin(p0[0]);
          s[2 * rr + 1] = dot_fin(p1[0]);
          ++jR;
          if (++slotR == nslot) { slotR = 0; phaseR ^= 1u; }
        }
      }
      const T tot = warp_multi_sum<K>(s, lane);   // lane (q << (5-LGK)) holds value q
#ifdef GF_FUSED_TRACE
      long long c0 = clock64();
#endif
      if (useR >= 1) mbar_wait_u32(rede0 + 8u * bR, (useR - 1) & 1u);
#ifdef GF_FUSED_TRACE
      if (tid == 0) GF_TR_ADD(9, c0);
#endif
      if (red_writer) red_dst[bR * (kFusedWarps * K)] = tot;
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(redf0 + 8u * bR);
      if (++bR == NE) { bR = 0; ++useR; }
    }
    if (t >= 2) {   // ---- C(t-2) ----
#ifdef GF_FUSED_TRACE
      long long c0 = clock64();
#endif
      mbar_wait_u32(wf0 + 8u * bC, useC & 1u);
#ifdef GF_FUSED_TRACE
      if (tid == 0) GF_TR_ADD(10, c0);
#endif
      T w0[TR], w1[TR];
#pragma unroll
      for (int rr = 0; rr < TR; ++rr) { w0[rr] = w_s[bC][rr][0]; w1[rr] = w_s[bC][rr][1]; }
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(we0 + 8u * bC);
      if (++bC == NE) { bC = 0; ++useC; }
#pragma unroll
      for (int rr = 0; rr < TR; ++rr) {
        if (jC < nr) {
          const uint32_t row = ring0 + (uint32_t)slotC * rb;
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const V a = lds128(row + voff[v], (V*)nullptr);
            vaxpy(ca[v], a, w0[rr]);
            vaxpy(cb[v], a, w1[rr]);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(sfree0 + 8u * slotC);
          ++jC;
          if (++slotC == nslot) slotC = 0;
        }
      }
    }
  }
  // column partials of this CTA (one slab)
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int64_t c = tid + (int64_t)v * kFusedThreads;
    if (c < nvec) {
      double* p0 = cpart + ((int64_t)blockIdx.x * 2) * ld + c * VN;
      double* p1 = cpart + ((int64_t)blockIdx.x * 2 + 1) * ld + c * VN;
#pragma unroll
      for (int i = 0; i < VN; ++i) {
        p0[i] = (double)vget(ca[v], i);
        p1[i] = (double)vget(cb[v], i);
      }
    }
  }
  }   // compute warps
  }   // consumer warps
  // every thread of an active CTA arrives here (the producer warp too; when
  // the solve has ended every CTA skips the tail alike)
  if (tail.on() && epi.active()) tail.run();
}


// ============================================================================
// Two-CTA cluster variant for wide rows (>= 40 KB: fp64 rows of 5000, fp32
// rows of 10000).  With whole rows only five fit in shared memory (one row
// per group: the serial epilogue then bounds the pass) and the compute warps
// would need 160 KB of register-resident column state.  Here the two CTAs of
// a cluster (two SMs) share one contiguous row range and split every row by
// columns: CTA r streams only its half of each row (TMA bulk copies of
// 20 KB), owns half of the column vectors (half the register state: the
// 8-warp x 5-vector shape of the fp32 n = 5000 kernel) and writes its
// half of the column slab.  Per group of TR rows the two CTAs exchange their
// K = 2 TR partial row dots through distributed shared memory -- the ONLY
// cross-SM hand-off: both then hold the full dots (summed as CTA 0's partial
// + CTA 1's, identical in both), both run the pure part of the epilogue
// (Epi::mid: the column-pass weights) for every row of the group, and row j's
// stores and reductions (Epi::tail) run in CTA (j & 1) only.  The weights
// hand-off to the compute warps stays CTA-local.
//
// The exchange uses st.async (asynchronous remote shared-memory stores that
// complete transaction bytes on the peer's mbarrier): no release fences, so
// the epilogue warp never waits for its own outstanding global stores (a
// release.cluster arrive compiles to MEMBAR.ALL.GPU), and the waits on it
// are CTA-scope (an acquire.cluster wait invalidates L1 every time).
// Buffers are double-buffered by use parity: xbuf[b][u & 1] / xf[b][u & 1]
// (count 1: the local arrive.expect_tx of K * 8 bytes; the peer's st.async
// completes them).  The peer can write use u + 2 only after it has received
// this CTA's partial of use u + 1, which is sent after use u was read -- so
// neither the slot nor the barrier phase can be overrun.
// A cluster barrier after the mbarrier init and one before exit keep every
// remote access inside both CTAs' lifetimes.
// ============================================================================

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> shared::cluster address of the same variable in CTA `rank`
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t addr, double v) { st_cluster_f64(addr, v); }
__device__ __forceinline__ void st_cluster(uint32_t addr, float v) { st_cluster_f32(addr, v); }
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster_u32(uint32_t bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(bar),
      "r"(parity), "r"(kSuspendNs)
      : "memory");
}

// st.async: 8-byte store into a peer CTA's shared memory that completes 8
// transaction bytes on the peer's mbarrier (both shared::cluster addresses).
__device__ __forceinline__ void st_async_f64(uint32_t cluster_addr, double v, uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(cluster_addr),
               "d"(v), "r"(cluster_bar)
               : "memory");
}
__device__ __forceinline__ void st_async_t(uint32_t cluster_addr, double v, uint32_t cluster_bar) {
  st_async_f64(cluster_addr, v, cluster_bar);
}
__device__ __forceinline__ void st_async_t(uint32_t cluster_addr, float v, uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(cluster_addr),
               "f"(v), "r"(cluster_bar)
               : "memory");
}

struct FusedPlan2 {
  int cl = 0;          // CTAs per cluster (2, 4 or 8): each streams 1/cl of every row
  int lag = 0;         // > 0: column pass on rows re-read from L2, lag groups behind (nslotc C-ring slots)
  int nslotc = 0;
  int cw = 0, ne = 0, nv = 0, nslot = 0, tr = 0;
  int grid = 0;        // CTAs (cl per cluster)
  int64_t hvec = 0;    // 16-byte vectors of the widest share of a row (the slot size)
  size_t smem = 0;
  bool ok = false;
};

// share of a row that CTA `rank` of a cl-CTA cluster streams: 16-byte vectors [v0, v1)
__host__ __device__ inline int64_t cl_vec_begin(int64_t nvec, int rank, int cl) { return nvec * rank / cl; }

// max_clusters: co-resident cl-CTA clusters at this shared-memory size
// (cudaOccupancyMaxActiveClusters): the kernel is persistent, every cluster
// must be resident in one wave.
inline FusedPlan2 plan_fused_cl(int64_t m, int64_t ld, int esize, int sms, size_t smem_max, int max_clusters, int cl,
                                int max_slots = kMaxSlots, int lag = 0) {
  FusedPlan2 p;
  p.cl = cl;
  p.lag = lag;
  const int vn = 16 / esize;
  const int64_t nvec = ld / vn;
  p.hvec = ceil_div(nvec, (int64_t)cl);
  p.cw = 20;
  for (int cw : {8, 12, 16, 20})
    if (ceil_div(p.hvec, cw * 32) <= (cw <= 12 ? 5 : 4)) { p.cw = cw; break; }
  p.nv = (int)ceil_div(p.hvec, p.cw * 32);
  p.ne = fused_epi_lag(p.cw, lag);
  const size_t slot_bytes = (size_t)p.hvec * 16;
  const size_t budget = smem_max > kStaticSmemReserve ? smem_max - kStaticSmemReserve : 0;
  p.nslot = (int)std::min<size_t>(std::min(max_slots, kMaxSlots), budget / slot_bytes);
  const int want_pf = std::max<int>(2, (int)ceil_div(48 * 1024, (int64_t)slot_bytes));
  p.tr = 0;
  if (lag > 0) {   // two rows per group; C ring: the group being read + one prefetched; R ring: the rest
    p.tr = 2;
    p.nslotc = 4;   // (6 measured the same on C2)
    p.nslot -= p.nslotc;
    if (p.nslot < p.tr + 2) p.tr = 0;
  } else
  for (int tr : {4, 2, 1})   // (2 TR (cl - 1) partials per group go out on distinct lanes)
    if ((3 * tr + want_pf <= p.nslot || (tr == 1 && 3 + 1 <= p.nslot)) && 2 * tr * (cl - 1) <= 32) {
      p.tr = tr;
      break;
    }
  const int64_t ncl = std::max<int64_t>(1, std::min<int64_t>({(int64_t)sms / cl, (int64_t)max_clusters, m}));
  p.grid = (int)(cl * ncl);
  p.smem = (size_t)(p.nslot + p.nslotc) * slot_bytes;
  // every CTA needs a non-empty share
  const bool shares = nvec >= cl && cl_vec_begin(nvec, 1, cl) >= 1;
  p.ok = max_clusters >= 1 && shares && p.nv >= 1 && p.nv <= 6 && p.tr >= 1 && m > 0 &&
         (cl == 2 || p.cw == 8) &&   // (the 4- and 8-CTA instances exist for 8 compute warps,
         (lag == 0 || (cl == 2 && p.cw == 8));   //  the lagged one for 2-CTA clusters of 8)
  return p;
}

// CL CTAs per cluster (2, 4, 8; the cluster shape is a launch attribute).
//
// LAG > 0 (heavy epilogues: Newton-prox losses): the column pass does not keep
// the rows in shared memory.  R(t) releases its slots at once; the producer
// re-reads the rows of group t - LAG from global memory (L2: the LAG groups
// of rows in between are a few tens of MB chip-wide) into a second ring, and
// C(t - LAG) runs on those.  Each CTA runs the epilogue of its own rows only
// and st.async-writes their weights into the peer too, and there are
// kLagEpi epilogue warps: a logistic prox is ~8 fp64 Newton steps, and the
// stream delivers ~1.2 rows per us per SM, so several rows must be in their
// Newton loop at once.  The weights live in a ring of LAG + 1 entries.
// nslot: R-ring slots; nslotc: C-ring slots (LAG > 0 only).

template <typename T, int NV, int TR, int CW, int CL, class Epi, class Tail = NoTail, int LAG = 0>
__global__ void __launch_bounds__(fused_threads_lag(CW, LAG), 1)
fused_rowcol_cl_kernel(const T* __restrict__ A, int64_t rows, int64_t ld, const T* __restrict__ x0,
                       const T* __restrict__ x1, Epi epi, int nslot, int64_t hvec, double* __restrict__ rpart,
                       double* __restrict__ cpart, Tail tail = Tail{}, int nslotc = 0) {
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
  constexpr int NR = Epi::NR;
  constexpr int K = 2 * TR;
  constexpr int LGK = K == 2 ? 1 : (K == 4 ? 2 : 3);
  constexpr int kFusedWarps = CW;
  constexpr int kFusedThreads = CW * kWarp;
  constexpr int NE = fused_epi_lag(CW, LAG);
  constexpr int kEpiWarp = CW;
  constexpr int kProdWarp = CW + NE;
  static_assert(CW <= 32, "one epilogue lane per compute warp");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxSlots], sfree[kMaxSlots];
  static_assert(CL == 2 || CL == 4 || CL == 8 || CL == 9, "cluster of 2, 4, 8 or 9 CTAs");
  static_assert(K * (CL - 1) <= 32, "one lane per (value, peer) partial");
  constexpr int WR = LAG > 0 ? LAG + 1 : NE;   // weight buffers: group g uses w_s[g % WR]
  constexpr int CLAG = LAG > 0 ? LAG : 2;      // the column pass of group t - CLAG runs after R(t)
  __shared__ __align__(8) uint64_t redf[NE], rede[NE], wf[WR], we[WR], xf[NE][2];
  __shared__ __align__(8) uint64_t fullc[LAG > 0 ? kMaxSlots : 1], freec[LAG > 0 ? kMaxSlots : 1];
  __shared__ T red_s[NE][kFusedWarps][K];
  __shared__ __align__(8) T w_s[WR][TR][2];
  __shared__ __align__(8) double xbuf[NE][2][CL][K];   // [buffer][use parity][source rank][value]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_ctarank();
  const int64_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int64_t nvec_all = ld / VN;
  const int64_t v0 = cl_vec_begin(nvec_all, (int)rank, CL);      // first 16-byte vector of this CTA's share
  const int64_t nvec = cl_vec_begin(nvec_all, (int)rank + 1, CL) - v0;
  const unsigned sb = (unsigned)(hvec * 16);               // slot stride
  const unsigned cb = (unsigned)(nvec * 16);               // bytes copied per row
  const int64_t r0 = rows * cid / ncl;
  const int64_t r1 = rows * (cid + 1) / ncl;
  const int nr = (int)(r1 - r0);
  const int ng = (nr + TR - 1) / TR;

  if (tid == 0) {
    for (int s = 0; s < nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sfree[s], kFusedWarps);
    }
    for (int b = 0; b < NE; ++b) {
      mbar_init(&redf[b], kFusedWarps);
      mbar_init(&rede[b], 1);
      mbar_init(&xf[b][0], 1);
      mbar_init(&xf[b][1], 1);
    }
    for (int b = 0; b < WR; ++b) {
      mbar_init(&wf[b], 1);
      mbar_init(&we[b], kFusedWarps);
    }
    if constexpr (LAG > 0)
      for (int s = 0; s < nslotc; ++s) {
        mbar_init(&fullc[s], 1);
        mbar_init(&freec[s], kFusedWarps);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster_sync_all();   // the peer's barriers exist before any remote arrive

  if (warp == kProdWarp) {
    // ===================== producer warp =====================
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int pre = min(nslot, nr);
      for (int j = 0; j < pre; ++j) {
        mbar_arrive_expect_tx(&full[j], cb);
        if constexpr (LAG > 0) bulk_g2s_nohint(smem_raw + j * sb, A + (r0 + j) * ld + v0 * VN, cb, &full[j]);
        else bulk_g2s(smem_raw + j * sb, A + (r0 + j) * ld + v0 * VN, cb, &full[j], pol);
      }
      pdl_wait();
      pdl_trigger();
      if (!epi.active()) {
        for (int j = 0; j < pre; ++j) mbar_wait(&full[j], 0u);
      } else if constexpr (LAG == 0) {
        int slot = pre == nslot ? 0 : pre;
        for (int j = pre; j < nr; ++j) {
          if (j >= nslot) mbar_wait(&sfree[slot], (unsigned)(((j / nslot) - 1) & 1));
          mbar_arrive_expect_tx(&full[slot], cb);
          bulk_g2s(smem_raw + slot * sb, A + (r0 + j) * ld + v0 * VN, cb, &full[slot], pol);
          if (++slot == nslot) slot = 0;
        }
      } else {
        // R loads at normal L2 priority: the line is read again LAG groups
        // later, by lane 1's column-ring loads below
        int slot = pre == nslot ? 0 : pre;
        for (int j = pre; j < nr; ++j) {
          if (j >= nslot) mbar_wait(&sfree[slot], (unsigned)(((j / nslot) - 1) & 1));
          mbar_arrive_expect_tx(&full[slot], cb);
          bulk_g2s_nohint(smem_raw + slot * sb, A + (r0 + j) * ld + v0 * VN, cb, &full[slot]);
          if (++slot == nslot) slot = 0;
        }
      }
    }
    if constexpr (LAG > 0) {
      // lane 1: the column-ring re-loads (evict-first: their last use), on
      // their own so that waiting for a column slot never holds back the
      // HBM row stream.  (Lanes 0 and 1 diverge; both spin on try_wait.)
      // (the status is read after the dependency wait: read before it, it
      // can be the previous kernel's RUNNING while the compute warps see the
      // stop, and this lane would wait forever for column slots nobody frees)
      if (lane == 1) pdl_wait();
      if (lane == 1 && epi.active()) {
        const uint64_t pol = policy_evict_first();
        unsigned char* ringc = smem_raw + (size_t)nslot * sb;
        int slotc = 0;
        for (int jc = 0; jc < nr; ++jc) {
          if (jc >= nslotc) mbar_wait(&freec[slotc], (unsigned)(((jc / nslotc) - 1) & 1));
          mbar_arrive_expect_tx(&fullc[slotc], cb);
          bulk_g2s(ringc + slotc * sb, A + (r0 + jc) * ld + v0 * VN, cb, &fullc[slotc], pol);
          if (++slotc == nslotc) slotc = 0;
        }
      }
    }
    __syncwarp();
  } else if (warp >= kEpiWarp && warp < kEpiWarp + NE) {
    // ===================== epilogue warps =====================
    pdl_wait();
    if (epi.active()) {
      const int par = warp - kEpiWarp;
      const int b = par;
      epi.begin();
      double ered[NR > 0 ? NR : 1];
#pragma unroll
      for (int k = 0; k < (NR > 0 ? NR : 1); ++k) ered[k] = 0.0;
      unsigned eflags = 0;
      // lane l < K (CL - 1) sends value l % K to peer (rank + 1 + l / K) % CL
      const int sq = lane % K;
      const uint32_t speer = (rank + 1u + (uint32_t)(lane / K)) % (uint32_t)CL;
      const bool sender = lane < K * (CL - 1);
      const uint32_t xb_peer = mapa_u32(smem_u32(&xbuf[b][0][rank][sq]), speer);   // my slot in the peer's buffer
      const uint32_t xf_peer = mapa_u32(smem_u32(&xf[b][0]), speer);
      const uint32_t xf_loc = smem_u32(&xf[b][0]), redf_loc = smem_u32(&redf[b]);
      constexpr uint32_t kUseStride = (uint32_t)(CL * K * sizeof(double));   // xbuf[b][1] - xbuf[b][0]
      typename Epi::RowIn in{};
      if (lane < TR && par * TR + lane < nr) in = epi.load_in(r0 + par * TR + lane);
      for (int ge = par; ge < ng; ge += NE) {
        const unsigned use = (unsigned)(ge / NE), p = use & 1u;
        mbar_wait_u32(redf_loc, use & 1u);
        // the sending lanes (< K (CL - 1)) must all hold the totals: a
        // half-warp butterfly leaves lanes 16-31 with their own (zero) half
        constexpr int RW = (CW <= 16 && K * (CL - 1) <= 16) ? 16 : 32;
        double v[K];
#pragma unroll
        for (int q = 0; q < K; ++q) v[q] = lane < kFusedWarps ? (double)red_s[b][lane][q] : 0.0;
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&rede[b], 0);
#pragma unroll
        for (int q = 0; q < K; ++q)
#pragma unroll
          for (int o = RW / 2; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o, RW);
        // this CTA's partials -> slot [rank] of every peer's xbuf[b][p]
        double mine_q = v[0];
#pragma unroll
        for (int q = 1; q < K; ++q)
          if (sq == q) mine_q = v[q];
        if (sender) st_async_f64(xb_peer + p * kUseStride, mine_q, xf_peer + 8u * p);
        if (lane == 0) mbar_arrive_expect_tx(&xf[b][p], (unsigned)((CL - 1) * K * sizeof(double)));
        mbar_wait_u32(xf_loc + 8u * p, (use >> 1) & 1u);   // every peer's partials have landed
        const int g = min(TR, nr - ge * TR);
        double dots[2] = {0.0, 0.0};
#pragma unroll
        for (int rr = 0; rr < TR; ++rr)
          if (rr == lane) {   // rank order 0 .. CL-1 (this CTA's own partial in its place): the same sum everywhere
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int r = 0; r < CL; ++r) {
              const double p0 = r == (int)rank ? v[2 * rr] : xbuf[b][p][r][2 * rr];
              const double p1 = r == (int)rank ? v[2 * rr + 1] : xbuf[b][p][r][2 * rr + 1];
              d0 = r == 0 ? p0 : d0 + p0;
              d1 = r == 0 ? p1 : d1 + p1;
            }
            dots[0] = d0;
            dots[1] = d1;
          }
        // every row's weights are computed here (mid is pure: every CTA gets
        // the same values); tail() only for this CTA's rows (row j: CTA j mod CL)
        const bool mine = lane < g && ((ge * TR + lane) % CL == (int)rank);
        typename Epi::Mid md{};
        double w0 = 0.0, w1 = 0.0;
        const int gw = ge % WR;
        const unsigned wuse = (unsigned)(ge / WR);
        if constexpr (LAG == 0) {
          if (lane < g) md = epi.mid(in, dots, w0, w1);
          if (wuse >= 1) mbar_wait_u32(smem_u32(&we[gw]), (wuse - 1) & 1u);    // w_s[gw] consumed by C(ge - WR)
          if (lane < g) {
            w_s[gw][lane][0] = (T)w0;
            w_s[gw][lane][1] = (T)w1;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_expect_tx(&wf[gw], 0);
        } else {
          // own rows only; their weights also go to the peer's w_s[gw] by
          // st.async (wf[gw]: the local arrival + the peer's bytes).  The peer
          // writes group ge only after it has this CTA's partials of ge, sent
          // after R(ge), which follows C(ge - WR) in this CTA's compute warps:
          // the slot is free by construction.
          static_assert(CL == 2 && TR % 2 == 0, "lagged pass: 2-CTA clusters, even TR");
          if (mine) md = epi.mid(in, dots, w0, w1);
          if (wuse >= 1) mbar_wait_u32(smem_u32(&we[gw]), (wuse - 1) & 1u);
          if (mine) {
            w_s[gw][lane][0] = (T)w0;
            w_s[gw][lane][1] = (T)w1;
            const uint32_t peer = rank ^ 1u;
            const uint32_t pw = mapa_u32(smem_u32(&w_s[gw][lane][0]), peer);
            const uint32_t pf = mapa_u32(smem_u32(&wf[gw]), peer);
            st_async_t(pw, (T)w0, pf);
            st_async_t(pw + (uint32_t)sizeof(T), (T)w1, pf);
          }
          __syncwarp();
          int own = 0;   // the peer's rows of this group: g - own, two values each
#pragma unroll
          for (int rr = 0; rr < TR; ++rr) own += (rr < g && ((ge * TR + rr) % CL == (int)rank)) ? 1 : 0;
          if (lane == 0) mbar_arrive_expect_tx(&wf[gw], (unsigned)((g - own) * 2 * sizeof(T)));
        }
        if (mine) epi.tail(r0 + (int64_t)ge * TR + lane, in, dots, md, ered, eflags);
        const int jn = (ge + NE) * TR + lane;
        if (lane < TR && jn < nr) in = epi.load_in(r0 + jn);
      }
#pragma unroll
      for (int k = 0; k < NR; ++k) ered[k] = warp_sum(ered[k]);
      eflags = warp_or(eflags);
      if (lane == 0) {
        double* out = rpart + (NE * (int64_t)blockIdx.x + par) * (NR + 1);
        for (int k = 0; k < NR; ++k) out[k] = ered[k];
        out[NR] = (double)eflags;
      }
    } else if (lane == 0) {   // inactive: empty records keep the Z step's sums defined
      double* out = rpart + (NE * (int64_t)blockIdx.x + (warp - kEpiWarp)) * (NR + 1);
      for (int k = 0; k <= NR; ++k) out[k] = 0.0;
    }
    __syncwarp();
  } else {
    // ===================== compute warps =====================
    pdl_wait();
    if (epi.active()) {
      V xa[NV], xb[NV], ca[NV], cb2[NV];
      uint32_t voff[NV];
      {
        const V* xv0 = reinterpret_cast<const V*>(x0) + v0;
        const V* xv1 = reinterpret_cast<const V*>(x1) + v0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int c = tid + v * kFusedThreads;
          const bool ok = c < (int)nvec;
          voff[v] = (uint32_t)(ok ? c : (int)nvec - 1) * 16u;
          xa[v] = ok ? xv0[c] : V{};
          xb[v] = ok ? xv1[c] : V{};
          ca[v] = V{};
          cb2[v] = V{};
        }
      }
      const uint32_t ring0 = smem_u32(smem_raw);
      const uint32_t full0 = smem_u32(full);
      const uint32_t sfree0 = smem_u32(sfree);
      const uint32_t redf0 = smem_u32(redf), rede0 = smem_u32(rede), wf0 = smem_u32(wf), we0 = smem_u32(we);
      const bool red_writer = (lane & ((32 >> LGK) - 1)) == 0;
      T* const red_dst = &red_s[0][warp][lane >> (5 - LGK)];
      int slotR = 0, slotC = 0;
      unsigned phaseR = 0, phaseC = 0;
      int jR = 0, jC = 0;
      int bR = 0, bC = 0;
      unsigned useR = 0, useC = 0;
      const uint32_t ringc0 = ring0 + (uint32_t)nslot * sb;
      const uint32_t fullc0 = smem_u32(fullc), freec0 = smem_u32(freec);
      for (int t = 0; t < ng + CLAG; ++t) {
        if (t < ng) {   // ---- R(t) ----
          T s[K];
#pragma unroll
          for (int rr = 0; rr < TR; ++rr) {
            s[2 * rr] = 0;
            s[2 * rr + 1] = 0;
            if (jR < nr) {
              mbar_wait_u32(full0 + 8u * slotR, phaseR);
              const uint32_t row = ring0 + (uint32_t)slotR * sb;
              typename DotAcc<T>::type p0[NV], p1[NV];
#pragma unroll
              for (int v = 0; v < NV; ++v) {
                const V a = lds128(row + voff[v], (V*)nullptr);
                p0[v] = dot_acc(a, xa[v]);
                p1[v] = dot_acc(a, xb[v]);
              }
              if constexpr (LAG > 0) {   // the row is re-read from L2 for the column pass
                __syncwarp();
                if (lane == 0) mbar_arrive_u32(sfree0 + 8u * slotR);
              }
#pragma unroll
              for (int v = 1; v < NV; ++v) { p0[0] = dot_add(p0[0], p0[v]); p1[0] = dot_add(p1[0], p1[v]); }
              s[2 * rr] = dot_fin(p0[0]);
              s[2 * rr + 1] = dot_fin(p1[0]);
              ++jR;
              if (++slotR == nslot) { slotR = 0; phaseR ^= 1u; }
            }
          }
          const T tot = warp_multi_sum<K>(s, lane);
          if (useR >= 1) mbar_wait_u32(rede0 + 8u * bR, (useR - 1) & 1u);
          if (red_writer) red_dst[bR * (kFusedWarps * K)] = tot;
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(redf0 + 8u * bR);
          if (++bR == NE) { bR = 0; ++useR; }
        }
        if (t >= CLAG) {   // ---- C(t - CLAG) ----
          mbar_wait_u32(wf0 + 8u * bC, useC & 1u);
          T w0[TR], w1[TR];
#pragma unroll
          for (int rr = 0; rr < TR; ++rr) { w0[rr] = w_s[bC][rr][0]; w1[rr] = w_s[bC][rr][1]; }
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(we0 + 8u * bC);
          if (++bC == WR) { bC = 0; ++useC; }
#pragma unroll
          for (int rr = 0; rr < TR; ++rr) {
            if (jC < nr) {
              uint32_t row;
              if constexpr (LAG > 0) {
                mbar_wait_u32(fullc0 + 8u * slotC, phaseC);
                row = ringc0 + (uint32_t)slotC * sb;
              } else {
                row = ring0 + (uint32_t)slotC * sb;
              }
#pragma unroll
              for (int v = 0; v < NV; ++v) {
                const V a = lds128(row + voff[v], (V*)nullptr);
                vaxpy(ca[v], a, w0[rr]);
                vaxpy(cb2[v], a, w1[rr]);
              }
              __syncwarp();
              if (lane == 0) mbar_arrive_u32((LAG > 0 ? freec0 : sfree0) + 8u * slotC);
              ++jC;
              if constexpr (LAG > 0) {
                if (++slotC == nslotc) { slotC = 0; phaseC ^= 1u; }
              } else {
                if (++slotC == nslot) slotC = 0;
              }
            }
          }
        }
      }
      // this CTA's columns of the cluster's slab
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int64_t c = tid + (int64_t)v * kFusedThreads;
        if (c < nvec) {
          double* p0 = cpart + (cid * 2) * ld + (v0 + c) * VN;
          double* p1 = cpart + (cid * 2 + 1) * ld + (v0 + c) * VN;
#pragma unroll
          for (int i = 0; i < VN; ++i) {
            p0[i] = (double)vget(ca[v], i);
            p1[i] = (double)vget(cb2[v], i);
          }
        }
      }
    }
  }
  __syncthreads();
  cluster_sync_all();   // no CTA leaves while its peer may still access its shared memory
  if (tail.on() && epi.active()) tail.run();
}

}  // namespace gf
