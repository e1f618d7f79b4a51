// Fused single-pass ADMM row/column kernel (tall problems, rows that fit in
// shared memory).
//
// The reference reads A four times per iteration (two projection matvecs plus
// the two residual matvecs on a second, unscaled copy; solver.py:197-198,
// projection.py:121-122), and the plain restatement still needs two passes:
// y+ = A_hat x+ (row pass) and A_hat' [c_y, nu^] (column pass).  But c_y and
// nu^ of row i depend only on row i's own dot products, so the column pass can
// consume each row right after the row pass has produced its epilogue -- while
// the row is still on chip.  One iteration then streams A_hat from HBM once:
//
//   persistent CTA per SM, contiguous row range; a ring of NSLOT row slots in
//   shared memory filled by TMA bulk copies (cp.async.bulk, L2 evict_first,
//   one mbarrier per slot); rows are consumed in groups of TR:
//     1. row pass    every thread owns fixed 16-byte column vectors (x^ and
//                    x^_1/2 for them live in registers for the whole kernel)
//     2. reduce      warp shuffles + one shared-memory stage -> 2 dots per row
//     3. epilogue    one thread per row (different warps): the full y side of
//                    the iteration (YEpi: dual step, prox_f, nu^, c_y, partials)
//     4. column pass the same threads re-read the same columns of the group's
//                    rows from shared memory and accumulate A' [c_y, nu^] in
//                    registers
//     5. release     barrier, then thread 0 refills the group's slots with rows
//                    NSLOT ahead
//   At the end each CTA writes its column partials (one "slab" per CTA) and
//   its epilogue reduction partials; colreduce + y_scalars finish them.
#pragma once

#include "gf_common.cuh"
#include "gf_gemv.cuh"

namespace gf {

constexpr int kFusedThreads = 512;
constexpr int kFusedWarps = kFusedThreads / kWarp;
constexpr int kMaxSlots = 32;
constexpr int kMaxTR = 8;

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

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
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
__device__ __forceinline__ void vaxpy(float4& acc, const float4& a, float w) {
  acc.x = fmaf(a.x, w, acc.x);
  acc.y = fmaf(a.y, w, acc.y);
  acc.z = fmaf(a.z, w, acc.z);
  acc.w = fmaf(a.w, w, acc.w);
}
__device__ __forceinline__ void vaxpy(double2& acc, const double2& a, double w) {
  acc.x = fma(a.x, w, acc.x);
  acc.y = fma(a.y, w, acc.y);
}

struct FusedPlan {
  int nv = 0;        // 16-byte vectors per thread per row (template instance)
  int nslot = 0;     // rows resident in shared memory
  int tr = 0;        // rows per group
  int grid = 0;      // CTAs (one per SM)
  size_t smem = 0;   // dynamic shared memory bytes
  bool ok = false;
};

inline FusedPlan plan_fused(int64_t m, int64_t ld, int esize, int sms, size_t smem_max) {
  FusedPlan p;
  const int vn = 16 / esize;
  const int64_t nvec = ld / vn;
  p.nv = (int)ceil_div(nvec, kFusedThreads);
  const size_t row_bytes = (size_t)ld * esize;
  const size_t budget = smem_max > 8192 ? smem_max - 8192 : 0;
  p.nslot = (int)std::min<size_t>(kMaxSlots, budget / row_bytes);
  // two resident groups (row pass of t, column pass of t-1) + TMA prefetch
  p.tr = std::min(kMaxTR, std::max(1, (p.nslot - 2) / 2));
  if (2 * p.tr + 1 > p.nslot) p.tr = 0;
  p.grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, m));
  p.smem = (size_t)p.nslot * row_bytes;
  p.ok = p.nv >= 1 && p.nv <= 6 && p.nslot >= 2 && p.tr >= 1 && m > 0;
  return p;
}

// Warp roles: warps 0..15 stream the row and column passes; warp 16 is the
// epilogue warp (lane rr handles row rr of a group).  Software pipeline over
// groups of TR rows, two CTA barriers per group:
//
//   iteration t:  compute warps   R(t): dots of group t -> red_s
//                 epilogue warp   (inputs of group t were prefetched in t-1)
//   --- barrier A ---
//                 epilogue warp   reduce red_s, y-side epilogue of group t
//                                 -> w_s[t&1]; prefetch inputs of group t+1
//                 compute warps   C(t-1): column pass of group t-1 with
//                                 w_s[(t-1)&1] (overlaps the epilogue)
//   --- barrier B ---
//                 thread 0        refill the slots of group t-1 (rows NSLOT ahead)
//
// so the serial epilogue latency hides behind a column pass, and the ring
// holds two groups plus NSLOT - 2*TR rows of TMA prefetch.
constexpr int kFusedCTA = kFusedThreads + kWarp;

template <typename T, int NV, class Epi>
__global__ void __launch_bounds__(kFusedCTA, 1)
fused_rowcol_kernel(const T* __restrict__ A, int64_t rows, int64_t ld, const T* __restrict__ x0,
                    const T* __restrict__ x1, Epi epi, int nslot, int tr, double* __restrict__ rpart,
                    double* __restrict__ cpart) {
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
  constexpr int NR = Epi::NR;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxSlots];
  __shared__ double red_s[kFusedWarps][2 * kMaxTR];
  __shared__ T w_s[2][kMaxTR][2];

  if (!epi.active()) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool is_epi = warp == kFusedWarps;
  const int64_t nvec = ld / VN;
  const size_t row_bytes = (size_t)ld * sizeof(T);
  const int64_t r0 = rows * blockIdx.x / gridDim.x;   // contiguous, balanced row range
  const int64_t r1 = rows * (blockIdx.x + 1) / gridDim.x;
  const int64_t nrows = r1 - r0;
  const int64_t ngroups = (nrows + tr - 1) / tr;

  if (tid == 0) {
    for (int s = 0; s < nslot; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol = 0;
  if (tid == 0) {
    pol = policy_evict_first();
    for (int s = 0; s < nslot && s < nrows; ++s) {
      mbar_arrive_expect_tx(&full[s], (unsigned)row_bytes);
      bulk_g2s(smem_raw + (size_t)s * row_bytes, A + (r0 + s) * ld, (unsigned)row_bytes, &full[s], pol);
    }
  }
  V xa[NV], xb[NV], ca[NV], cb[NV];
  if (!is_epi) {
    const V* xv0 = reinterpret_cast<const V*>(x0);
    const V* xv1 = reinterpret_cast<const V*>(x1);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int64_t c = tid + (int64_t)v * kFusedThreads;
      xa[v] = c < nvec ? xv0[c] : V{};
      xb[v] = c < nvec ? xv1[c] : V{};
      ca[v] = V{};
      cb[v] = V{};
    }
  }
  double ered[NR > 0 ? NR : 1];
#pragma unroll
  for (int k = 0; k < (NR > 0 ? NR : 1); ++k) ered[k] = 0.0;
  unsigned eflags = 0;
  typename Epi::RowIn in_next{};
  if (is_epi && lane < tr && lane < nrows) in_next = epi.load_in(r0 + lane);

  for (int64_t t = 0; t <= ngroups; ++t) {
    const int64_t j0 = t * tr;
    const int g = t < ngroups ? (int)min((int64_t)tr, nrows - j0) : 0;
    if (!is_epi && g > 0) {
      // ---- R(t): row pass of group t ----
      T s0[kMaxTR], s1[kMaxTR];
#pragma unroll
      for (int rr = 0; rr < kMaxTR; ++rr) { s0[rr] = 0; s1[rr] = 0; }
#pragma unroll
      for (int rr = 0; rr < kMaxTR; ++rr) {
        if (rr < g) {
          const int64_t j = j0 + rr;
          const int slot = (int)(j % nslot);
          mbar_wait(&full[slot], (unsigned)((j / nslot) & 1));
          const V* row = reinterpret_cast<const V*>(smem_raw + (size_t)slot * row_bytes);
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const int64_t c = tid + (int64_t)v * kFusedThreads;
            if (c < nvec) {
              const V a = row[c];
              s0[rr] = vdot(a, xa[v], s0[rr]);
              s1[rr] = vdot(a, xb[v], s1[rr]);
            }
          }
        }
      }
#pragma unroll
      for (int rr = 0; rr < kMaxTR; ++rr) {
        if (rr < g) {
          const T a = warp_sum(s0[rr]);
          const T b = warp_sum(s1[rr]);
          if (lane == 0) {
            red_s[warp][2 * rr] = (double)a;
            red_s[warp][2 * rr + 1] = (double)b;
          }
        }
      }
    }
    __syncthreads();  // A
    if (is_epi) {
      if (lane < g) {   // ---- epilogue of group t ----
        const int rr = lane;
        double dots[2] = {0.0, 0.0};
        for (int w = 0; w < kFusedWarps; ++w) {
          dots[0] += red_s[w][2 * rr];
          dots[1] += red_s[w][2 * rr + 1];
        }
        double w0, w1;
        epi.finish(r0 + j0 + rr, in_next, dots, ered, eflags, w0, w1);
        w_s[t & 1][rr][0] = (T)w0;
        w_s[t & 1][rr][1] = (T)w1;
      }
      const int64_t jn = j0 + tr + lane;   // prefetch the inputs of group t+1
      if (lane < tr && jn < nrows) in_next = epi.load_in(r0 + jn);
    } else if (t >= 1) {
      // ---- C(t-1): column pass of the previous group ----
      const int64_t jp = j0 - tr;
      const int gp = (int)min((int64_t)tr, nrows - jp);
#pragma unroll
      for (int rr = 0; rr < kMaxTR; ++rr) {
        if (rr < gp) {
          const int slot = (int)((jp + rr) % nslot);
          const V* row = reinterpret_cast<const V*>(smem_raw + (size_t)slot * row_bytes);
          const T w0 = w_s[(t - 1) & 1][rr][0], w1 = w_s[(t - 1) & 1][rr][1];
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const int64_t c = tid + (int64_t)v * kFusedThreads;
            if (c < nvec) {
              const V a = row[c];
              vaxpy(ca[v], a, w0);
              vaxpy(cb[v], a, w1);
            }
          }
        }
      }
    }
    __syncthreads();  // B
    if (tid == 0 && t >= 1) {   // refill the slots of group t-1
      const int64_t jp = j0 - tr;
      const int gp = (int)min((int64_t)tr, nrows - jp);
      for (int rr = 0; rr < gp; ++rr) {
        const int64_t jn = jp + rr + nslot;
        if (jn < nrows) {
          const int slot = (int)(jn % nslot);
          mbar_arrive_expect_tx(&full[slot], (unsigned)row_bytes);
          bulk_g2s(smem_raw + (size_t)slot * row_bytes, A + (r0 + jn) * ld, (unsigned)row_bytes, &full[slot], pol);
        }
      }
    }
  }
  if (!is_epi) {   // column partials of this CTA (one slab)
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
  } else {         // epilogue partials, held by the epilogue warp
#pragma unroll
    for (int k = 0; k < NR; ++k) ered[k] = warp_sum(ered[k]);
    eflags = warp_or(eflags);
    if (lane == 0) {
      for (int k = 0; k < NR; ++k) rpart[blockIdx.x * (NR + 1) + k] = ered[k];
      rpart[blockIdx.x * (NR + 1) + NR] = (double)eflags;
    }
  }
}

}  // namespace gf
