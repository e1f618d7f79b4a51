// G^-1 GEMV with the x-side epilogue on a TMA row ring (tall iterations,
// S step: x+ = G^-1 rhs, then prox_g etc. per column, projection.py:121 and
// solver.py:330-335, 393, 419).
//
// The plain row GEMV (one warp per row, loads in a loop) is latency-bound for
// G^-1: each warp owns ~2 rows of 20 KB and its trip count is the latency
// chain.  Here, like the fused pass, one persistent CTA per SM streams its
// contiguous block of rows through a ring of shared-memory slots filled by
// TMA bulk copies (a producer warp, the first fill issued before the
// programmatic-dependency wait since G^-1 is constant); CW compute warps
// hold fixed column vectors of rhs in registers and produce one partial dot
// per row and warp; an epilogue warp adds the CW partials of 32 rows at a time
// (fixed order, fp64) and runs Epi::row for those rows on its 32 lanes in
// parallel.  Hand-offs are mbarriers; partial buffers are double-buffered.
#pragma once

#include "gf_fused.cuh"

namespace gf {

struct RingPlan {
  int cw = 0, nv = 0, nslot = 0, grid = 0;
  size_t smem = 0;
  bool ok = false;
};

inline RingPlan plan_ring(int64_t rows, int64_t ld, int esize, int sms, size_t smem_max, int64_t max_grid) {
  RingPlan p;
  const int64_t nvec = ld / (16 / esize);
  p.cw = 20;
  for (int cw : {8, 12, 16, 20})
    if (ceil_div(nvec, cw * 32) <= (cw <= 12 ? 5 : 4)) { p.cw = cw; break; }
  p.nv = (int)ceil_div(nvec, p.cw * 32);
  const size_t row_bytes = (size_t)ld * esize;
  if (row_bytes == 0) return p;
  const size_t budget = smem_max > 16384 ? smem_max - 16384 : 0;
  p.nslot = (int)std::min<size_t>(16, budget / row_bytes);
  p.grid = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)sms, rows, max_grid}));
  p.smem = (size_t)p.nslot * row_bytes;
  p.ok = rows > 0 && p.nslot >= 4 && p.nv >= 1 && p.nv <= (p.cw <= 12 ? 5 : 4);
  return p;
}

template <typename T, int NV, int CW, class Epi>
__global__ void __launch_bounds__((CW + 2) * 32, 1)
ring_gemv_kernel(const T* __restrict__ A, int64_t rows, int64_t ld, const T* __restrict__ x, Epi epi, int nslot,
                 double* __restrict__ part, int64_t npart) {
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
  constexpr int NR = Epi::NR;
  constexpr int kEpiWarp = CW, kProdWarp = CW + 1, kThreads = CW * 32;
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[kMaxSlots], sfree[kMaxSlots], redf[2], rede[2];
  __shared__ T red[2][CW][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  const int nr = (int)(r1 - r0);
  const unsigned rb = (unsigned)(ld * sizeof(T));
  if (tid == 0) {
    for (int s = 0; s < nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sfree[s], CW);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&redf[b], CW);
      mbar_init(&rede[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kProdWarp) {
    // ===================== producer warp =====================
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int pre = min(nslot, nr);
      for (int j = 0; j < pre; ++j) {
        mbar_arrive_expect_tx(&full[j], rb);
        bulk_g2s(ring + j * rb, A + (r0 + j) * ld, rb, &full[j], pol);
      }
      pdl_wait();
      pdl_trigger();
      if (!epi.active()) {
        for (int j = 0; j < pre; ++j) mbar_wait(&full[j], 0u);
        return;
      }
      int slot = pre == nslot ? 0 : pre;
      for (int j = pre; j < nr; ++j) {
        mbar_wait(&sfree[slot], (unsigned)(((j / nslot) - 1) & 1));
        mbar_arrive_expect_tx(&full[slot], rb);
        bulk_g2s(ring + slot * rb, A + (r0 + j) * ld, rb, &full[slot], pol);
        if (++slot == nslot) slot = 0;
      }
    }
    return;
  }
  pdl_wait();
  if (!epi.active()) return;

  if (warp == kEpiWarp) {
    // ===================== epilogue warp =====================
    // records this grid does not produce are zero (the Z step sums npart)
    for (int64_t i = (int64_t)gridDim.x * (NR + 1) + (int64_t)blockIdx.x * 32 + lane; i < npart * (NR + 1);
         i += (int64_t)gridDim.x * 32)
      part[i] = 0.0;
    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int k = 0; k < (NR > 0 ? NR : 1); ++k) acc[k] = 0.0;
    unsigned flags = 0;
    const int nbatch = (nr + 31) / 32;
    for (int t = 0; t < nbatch; ++t) {
      const int b = t & 1;
      mbar_wait(&redf[b], (unsigned)((t >> 1) & 1));
      const int cnt = min(32, nr - t * 32);
      double sum = 0.0;
      if (lane < cnt)
#pragma unroll
        for (int w = 0; w < CW; ++w) sum += (double)red[b][w][lane];
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&rede[b], 0);   // red[b] may be rewritten
      if (lane < cnt) {
        const double dots[2] = {sum, 0.0};
        epi.row(r0 + (int64_t)t * 32 + lane, dots, acc, flags);
      }
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) acc[k] = warp_sum(acc[k]);
    flags = warp_or(flags);
    if (lane == 0) {
      double* out = part + (int64_t)blockIdx.x * (NR + 1);
      for (int k = 0; k < NR; ++k) out[k] = acc[k];
      out[NR] = (double)flags;
    }
    return;
  }

  // ===================== compute warps =====================
  V xa[NV];
  uint32_t voff[NV];
  {
    const int64_t nvec = ld / VN;
    const V* xv = reinterpret_cast<const V*>(x);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = tid + v * kThreads;
      const bool ok = c < (int)nvec;
      voff[v] = (uint32_t)(ok ? c : (int)nvec - 1) * 16u;   // clamped: zero x adds exact zeros
      xa[v] = ok ? xv[c] : V{};
    }
  }
  const uint32_t ring0 = smem_u32(ring), full0 = smem_u32(full), sfree0 = smem_u32(sfree);
  const uint32_t redf0 = smem_u32(redf), rede0 = smem_u32(rede);
  int slot = 0;
  unsigned phase = 0;
  for (int j = 0; j < nr; ++j) {
    mbar_wait_u32(full0 + 8u * slot, phase);
    const uint32_t row = ring0 + (uint32_t)slot * rb;
    typename DotAcc<T>::type p[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) p[v] = dot_acc(lds128(row + voff[v], (V*)nullptr), xa[v]);
#pragma unroll
    for (int v = 1; v < NV; ++v) p[0] = dot_add(p[0], p[v]);
    const T d = warp_sum(dot_fin(p[0]));
    __syncwarp();
    if (lane == 0) mbar_arrive_u32(sfree0 + 8u * slot);
    if (++slot == nslot) { slot = 0; phase ^= 1u; }
    const int t = j >> 5, b = t & 1;
    if ((j & 31) == 0 && t >= 2) mbar_wait_u32(rede0 + 8u * b, (unsigned)(((t >> 1) - 1) & 1));
    if (lane == 0) red[b][warp][j & 31] = d;
    if ((j & 31) == 31 || j == nr - 1) {
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(redf0 + 8u * b);
    }
  }
}

}  // namespace gf
