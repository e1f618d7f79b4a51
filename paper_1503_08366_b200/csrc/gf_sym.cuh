// G^-1 GEMV on the lower triangle only, with the x-side epilogue (tall
// iterations, S step: x+ = G^-1 rhs then prox_g etc. per column,
// projection.py:121, solver.py:330-335, 393, 419).
//
// G^-1 = (I + A_hat' A_hat)^-1 is symmetric, so half of it carries all the
// information: each 64 x 64 tile (I, J), J <= I, of the lower triangle is
// read from HBM once and used twice -- y_I += G_IJ x_J and, off the
// diagonal, y_J += G_IJ' x_I.  The projection's bytes per iteration halve
// (q^2/2 elements instead of q^2: 50 MB instead of 100 MB at q = 5000 fp32,
// 1.6 GB instead of 3.2 GB at C3's q = 20000 fp64).
//
// One persistent CTA per SM takes a contiguous range of the tiles in
// row-block order; a producer warp streams them through a ring of shared-
// memory slots with 2-D TMA loads (the first fill issued before the
// programmatic-dependency wait: G^-1 is constant), and compute warp w of W
// processes the CTA's tiles w, w + W, ...: lane l owns columns 2l, 2l + 1 of
// the tile, accumulates the column partials over its 64 rows and per-lane
// row partials, 32 rows at a time, which a butterfly reduce-scatter turns
// into one row sum per lane.  Every tile writes its 64 row and 64 column
// partials (fp64) to a scratch array -- no atomics.  After a grid barrier CTA
// b finishes columns [q b/G, q (b+1)/G): y_j is the sum of the nb partials of
// block K = j / 64 (row partials of tiles (K, 0..K), then column partials of
// tiles (K+1..nb-1, K)), in a fixed order, and the x side runs on it.  Every
// sum has a fixed order: the result is the same on every run and every rank.
#pragma once

#include <cuda.h>

#include "gf_fused.cuh"

namespace gf {

constexpr int kSymTB = 64;       // tile edge
// Compute warps (also the phase-2 warps): at most the ring's slot count --
// warp w waits on tile j's slot with parity (j / nslot) & 1, which is only
// unambiguous when the slot's previous tile j - nslot is already loaded,
// i.e. when nslot >= the number of warps taking tiles round-robin.  fp64
// tiles are 32 KB: 6 slots, 6 warps.
template <typename T>
__host__ __device__ constexpr int sym_warps() { return sizeof(T) == 8 ? 6 : 8; }
template <typename T>
__host__ __device__ constexpr int sym_threads() { return (sym_warps<T>() + 1) * 32; }
constexpr int kSymBatch = 10;    // phase 2: partial loads in flight per lane

struct SymPlan {
  int nslot = 0, grid = 0;
  int64_t nb = 0, nt = 0;   // row blocks, lower-triangle tiles
  size_t smem = 0;
  bool ok = false;
};

inline SymPlan plan_sym(int64_t q, int64_t ldq, int esize, int sms, size_t smem_max, int64_t max_grid) {
  const int warps = esize == 8 ? sym_warps<double>() : sym_warps<float>();
  SymPlan p;
  p.nb = ceil_div(q, (int64_t)kSymTB);
  p.nt = p.nb * (p.nb + 1) / 2;
  const size_t tile = (size_t)kSymTB * kSymTB * esize;
  const size_t budget = smem_max > 16384 ? smem_max - 16384 : 0;
  p.nslot = (int)std::min<size_t>(12, budget / tile);
  // a multiple of the warp count: tile j goes to warp j % W and slot
  // j % nslot, so every slot then belongs to one warp, which waits on its
  // phases in order.  With slots shared by several warps (12 slots, 8 warps:
  // the fp32 plan before) a warp running ahead of a slow one can match a
  // phase of the same parity two rounds old, consume a stale tile and
  // release its slot early -- the intermittent stall of DESIGN §4.
  p.nslot -= p.nslot % warps;
  p.grid = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)sms, p.nt, max_grid}));
  p.smem = (size_t)p.nslot * tile;
  p.ok = q >= kSymTB && p.nslot >= warps && (ldq * esize) % 16 == 0;
  return p;
}

// tile t of the row-block-major lower triangle -> (I, J), J <= I
__device__ __forceinline__ void sym_tile(int64_t t, int64_t& I, int64_t& J) {
  int64_t i = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (i * (i + 1) / 2 > t) --i;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  I = i;
  J = t - i * (i + 1) / 2;
}

__device__ __forceinline__ int64_t sym_index(int64_t I, int64_t J) { return I * (I + 1) / 2 + J; }

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
      "{%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}

template <typename T>
struct SymPair;
template <>
struct SymPair<float> {
  using type = float2;
};
template <>
struct SymPair<double> {
  using type = double2;
};

// Grid barrier on its own counters (gf_solver.cu's Ctl::scnt / sgen).
__device__ __forceinline__ void sym_grid_sync(unsigned* cnt, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vg = gen;
    const unsigned g0 = *vg;
    __threadfence();
    if (atomicAdd(cnt, 1u) == gridDim.x - 1) {
      atomicExch(cnt, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vg == g0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

template <typename T, class Epi>
__global__ void __launch_bounds__(sym_threads<T>(), 1)
sym_gemv_kernel(const __grid_constant__ CUtensorMap tm, int64_t q, const T* __restrict__ x, Epi epi, int nslot,
                int64_t nb, int64_t nt, double* __restrict__ spart, unsigned* gcnt, unsigned* ggen,
                double* __restrict__ part, int64_t npart) {
  using P2 = typename SymPair<T>::type;
  constexpr int kSymWarps = sym_warps<T>();
  constexpr int NR = Epi::NR;
  constexpr int TB = kSymTB;
  constexpr unsigned kTileBytes = (unsigned)(TB * TB * sizeof(T));
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[16], sfree[16];
  __shared__ T xs[kSymWarps][TB];
  __shared__ double comb[kSymWarps][33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t t0 = nt * b / G, t1 = nt * (b + 1) / G;
  const int ntl = (int)(t1 - t0);
  if (tid == 0) {
    for (int s = 0; s < nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sfree[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kSymWarps) {
    // ===================== producer warp (phase 1) =====================
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int pre = min(nslot, ntl);
      for (int j = 0; j < pre; ++j) {
        int64_t I, J;
        sym_tile(t0 + j, I, J);
        mbar_arrive_expect_tx(&full[j], kTileBytes);
        tma_load_2d(smem_u32(ring + (size_t)j * kTileBytes), &tm, (int)(J * TB), (int)(I * TB), smem_u32(&full[j]),
                    pol);
      }
      pdl_wait();
      pdl_trigger();
      if (epi.active()) {
        int slot = pre == nslot ? 0 : pre;
        for (int j = pre; j < ntl; ++j) {
          int64_t I, J;
          sym_tile(t0 + j, I, J);
          mbar_wait(&sfree[slot], (unsigned)(((j / nslot) - 1) & 1));
          mbar_arrive_expect_tx(&full[slot], kTileBytes);
          tma_load_2d(smem_u32(ring + (size_t)slot * kTileBytes), &tm, (int)(J * TB), (int)(I * TB),
                      smem_u32(&full[slot]), pol);
          if (++slot == nslot) slot = 0;
        }
      } else {
        for (int j = 0; j < pre; ++j) mbar_wait(&full[j], 0u);
      }
    }
  } else {
    pdl_wait();
    if (epi.active()) {
      // ===================== compute warps (phase 1) =====================
      for (int j = warp; j < ntl; j += kSymWarps) {
        const int slot = j % nslot;
        int64_t I, J;
        sym_tile(t0 + j, I, J);
        const int64_t ci = J * TB + 2 * lane, ri = I * TB + 2 * lane;
        const double xj0 = ci < q ? (double)x[ci] : 0.0, xj1 = ci + 1 < q ? (double)x[ci + 1] : 0.0;
        xs[warp][2 * lane] = ri < q ? x[ri] : (T)0;
        xs[warp][2 * lane + 1] = ri + 1 < q ? x[ri + 1] : (T)0;
        __syncwarp();
        mbar_wait(&full[slot], (unsigned)((j / nslot) & 1));
        const unsigned char* tile = ring + (size_t)slot * kTileBytes;
        const T xa = (T)xj0, xb = (T)xj1;
        T c0 = (T)0, c1 = (T)0;
        double* out = spart + (t0 + j) * (2 * TB);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          T rp[32];
#pragma unroll
          for (int rr = 0; rr < 32; ++rr) {
            const int r = h * 32 + rr;
            const P2 a = *reinterpret_cast<const P2*>(tile + ((size_t)r * TB + 2 * lane) * sizeof(T));
            const T xr = xs[warp][r];
            rp[rr] = fma(a.x, xa, a.y * xb);
            c0 = fma(a.x, xr, c0);
            c1 = fma(a.y, xr, c1);
          }
          // reduce-scatter: lane l ends with the sum over the 32 lanes of row h*32 + l
#pragma unroll
          for (int o = 16, n = 16; o >= 1; o >>= 1, n >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int k = 0; k < n; ++k) {
              const T send = up ? rp[k] : rp[k + n];
              const T keep = up ? rp[k + n] : rp[k];
              rp[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          out[h * 32 + lane] = (double)rp[0];
        }
        out[TB + 2 * lane] = I > J ? (double)c0 : 0.0;
        out[TB + 2 * lane + 1] = I > J ? (double)c1 : 0.0;
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(smem_u32(&sfree[slot]));
      }
    }
  }
  if (!epi.active()) return;

  // ===================== phase 2: the columns of this CTA =====================
  sym_grid_sync(gcnt, ggen);
  // records this grid does not produce are zero (the Z step sums npart)
  if (tid < 32)
    for (int64_t i = G * (NR + 1) + b * 32 + tid; i < npart * (NR + 1); i += G * 32) part[i] = 0.0;
  const int64_t c0 = q * b / G, c1 = q * (b + 1) / G;
  double acc[NR > 0 ? NR : 1];
#pragma unroll
  for (int k = 0; k < (NR > 0 ? NR : 1); ++k) acc[k] = 0.0;
  unsigned flags = 0;
  for (int64_t cc = c0; cc < c1; cc += 32) {   // uniform trip count in the CTA
    const int64_t jc = cc + lane;
    double s = 0.0;
    if (warp < kSymWarps && jc < c1) {
      const int64_t K = jc / TB;
      const int e = (int)(jc % TB);
      // warp w: terms u = w, w + W, ... (u <= K: row partial of tile (K, u);
      // u > K: column partial of tile (u, K)), loads batched, summed in order
      for (int64_t u0 = warp; u0 < nb; u0 += (int64_t)kSymWarps * kSymBatch) {
        double v[kSymBatch];
#pragma unroll
        for (int k = 0; k < kSymBatch; ++k) {
          const int64_t u = u0 + (int64_t)kSymWarps * k;
          v[k] = u >= nb ? 0.0
                         : (u <= K ? spart[sym_index(K, u) * (2 * TB) + e]
                                   : spart[sym_index(u, K) * (2 * TB) + TB + e]);
        }
#pragma unroll
        for (int k = 0; k < kSymBatch; ++k) s += v[k];
      }
    }
    if (warp < kSymWarps) comb[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && jc < c1) {
      double y = comb[0][lane];
#pragma unroll
      for (int w = 1; w < kSymWarps; ++w) y += comb[w][lane];
      const double dots[2] = {y, 0.0};
      epi.row(jc, dots, acc, flags);
    }
    __syncthreads();
  }
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < NR; ++k) acc[k] = warp_sum(acc[k]);
    flags = warp_or(flags);
    if (lane == 0) {
      double* o = part + b * (NR + 1);
      for (int k = 0; k < NR; ++k) o[k] = acc[k];
      o[NR] = (double)flags;
    }
  }
}

}  // namespace gf
