// Tensor-core Gram matrix G = A'A for fp32 A (tall projector setup) on
// tcgen05 with a three-product split for fp32-grade accuracy.
//
// Reference: projection.py:86-90 (gram = A.T @ A; gram += I) on OpenBLAS dgemm.
// The north star asks for a tensor-core SYRK; plain TF32 perturbs G enough to
// move fp32 iterates (x error 3.5e-4 on SVM) and BF16 changes
// iteration counts, so each fp32 element is split as a = hi + lo and
//     G += hi_i' hi_j + hi_i' lo_j + lo_i' hi_j           (3 MMAs)
// which keeps ~22 mantissa bits.  Default split (kind::f16): the panel is
// scaled by a power of two s (largest entry ~2^14) and hi = f16(s a),
// lo = f16(s a - hi); the drain multiplies by 1/s^2.  GF_SYRK=tf32 selects
// the kind::tf32 split hi = tf32(a), lo = tf32(a - hi), which moves twice the
// operand bytes per MAC (Gram 26.5 -> 23.6 ms at 200000 x 5000 for f16).
// The accumulator lives in TMEM in fp32 and is drained into the fp64 G every
// `kchunk` rows: the tensor core's fp32 accumulation truncates, so its
// relative error grows with the number of accumulate steps per drain
// (measured ~3e-8 per step); the drain interval bounds it while the long
// reduction over m = 2e5 rows is carried in fp64.
//
// Tile: 128 columns of A (MMA M) x 256 columns (MMA N), lower-triangle tiles
// only (G is mirrored afterwards).  Warp roles (576 threads):
//   warps 0-3   epilogue: tcgen05.ld the 128x256 fp32 accumulator, add into G (fp64)
//   warp 4      TMEM allocator + MMA issuer (one thread)
//   warps 5-16  converters: column reads of the raw TMA slab, split into
//               hi/lo, one 16-byte store each into the K-major no-swizzle
//               core-matrix layout the MMA descriptors expect
//   warp 17     TMA loader (2-D tensor maps, raw fp32 ring)
// Pipelines: raw ring (TMA -> converters), operand stages (full/empty
// mbarriers; empty is signalled by tcgen05.commit) and 2 TMEM accumulators
// (256 columns each; full by tcgen05.commit, empty by the epilogue warps).
//
// What bounds it is shared-memory bandwidth: per 16-row stage the TMA writes
// 24 KB, the converters read 24 KB and write 24 KB (f16) and the three MMAs
// read 36 KB -- ~860 wavefronts against 384 tensor-pipe cycles.  Measured by
// switching parts off: conversion alone 18.5 ms, MMA alone 14.4 ms, all
// 24.5 ms (the costs add); drain interval, barrier polling back-off and an
// L2 evict-last policy on the G tiles made no difference.

#include <cuda.h>
#include <chrono>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "gf_internal.h"

namespace gf {
namespace syrk {

// K-major, no-swizzle operand layout (verified on B200 with tools/umma_probe.cu):
// a core matrix is 8 MN-rows x 16 bytes (4 tf32 along K), 128 contiguous
// bytes; 8-row groups are SBO = 128 B apart, 4-element K chunks LBO apart.
constexpr int TM = 128, TN = 256, BK = 16;
// rows per TMEM accumulation: 1024 -> max |G error| / max |G| ~ 9.5e-6 on a
// 20000 x 1300 Gaussian matrix (512: 4.7e-6, 128: 1.2e-6; tools/syrk_accuracy.py);
// 1024 halves the fp64 drain traffic of 512 (Gram 39 -> 29 ms at 200000 x 5000)
constexpr int KCHUNK_DEFAULT = 1024;
constexpr int NPROD = 12;                          // converter warps
constexpr int LOADER_WARP = 5 + NPROD;             // TMA loader warp
constexpr int THREADS = (6 + NPROD) * 32;
// raw fp32 ring filled by 2-D tensor TMA: per stage two boxes, BK rows x TM
// columns (A panel, 8 KB) then BK rows x TN columns (B panel, 16 KB), rows
// and columns past the matrix zero-filled by the TMA unit
constexpr int RAW_A = BK * TM * 4;
constexpr int RAW_BYTES = BK * (TM + TN) * 4;      // 24 KB
constexpr int NRAW = 5;

// Operand split.  F16 = false: tf32 hi/lo (4-byte elements, 4 per core-matrix
// row, K = 8 per MMA).  F16 = true: the panel is scaled by s = 2^(14 - e_max)
// (exact) and split into fp16 hi/lo (2-byte elements, 8 per core-matrix row,
// K = 16 per MMA at twice the tf32 rate); the drain multiplies by 1/s^2.
// Same 11 + 11 mantissa bits as 3xTF32; fp16's exponent range is what the
// scale is for (entries below 2^-24 of the largest lose bits in absolute terms
// only, ~2^-25 max|A| per element).  Half the operand bytes per MAC: the
// shared-memory traffic per K row drops from 1350 to ~880 B-cycles.
template <bool F16>
struct Split {
  static constexpr int ESZ = F16 ? 2 : 4;
  static constexpr int KCH = 16 / ESZ;             // K elements per core-matrix row
  static constexpr int A_BYTES = BK * TM * ESZ;    // per hi/lo
  static constexpr int B_BYTES = BK * TN * ESZ;
  static constexpr int LBO_A = (TM / 8) * 128;     // K-chunk stride
  static constexpr int LBO_B = (TN / 8) * 128;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;   // 48 / 24 KB
  static constexpr int NST = F16 ? 4 : 2;
  static constexpr int KSTEPS = BK / (2 * KCH);    // MMAs (x3) per stage: 2 / 1
  static constexpr int SMEM = NST * STAGE + NRAW * RAW_BYTES;   // 96 + 120 KB
  // Instruction descriptor: D f32, A/B tf32 (2) or f16 (0), K-major, M = 128, N = 256.
  static constexpr uint32_t IDESC = (1u << 4) | ((F16 ? 0u : 2u) << 7) | ((F16 ? 0u : 2u) << 10) |
                                    ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// Shared-memory matrix descriptor: no swizzle, Blackwell version 1.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
  return d;                 // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

template <bool F16>
__device__ __forceinline__ void mma_split(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  if constexpr (F16)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(Split<F16>::IDESC), "r"(accumulate));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(Split<F16>::IDESC), "r"(accumulate));
}

__device__ __forceinline__ uint32_t pack_f16(float a, float b) {   // a -> low half (lower K index)
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// scale exponent: s = 2^(14 - e), e = exponent of max|A| (bits of the float max)
__device__ __forceinline__ int split_shift(const unsigned* amax_bits) {
  const unsigned b = amax_bits ? *amax_bits : 0u;
  if (b == 0u || b >= 0x7f800000u) return 0;
  const int e = (int)(b >> 23) - 127;   // max|A| in [2^e, 2^(e+1))
  return min(126, max(-126, 14 - e));
}

__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
               : "memory");
}

// Epilogue warp `warp` (0-3) adds its 32 TMEM lanes (tile rows i) of
// accumulator `acc` into G, scaled by `unscale`.
__device__ __forceinline__ void drain_chunk(uint32_t tmem, int warp, int acc, int64_t i, int64_t j0, int64_t q,
                                            double* __restrict__ G, int64_t ldg, double unscale) {
#pragma unroll 1
  for (int cc = 0; cc < TN / 16; ++cc) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * TN + cc * 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    // G is symmetric: accumulate the tile's transpose, G[j][i], so the 32
    // lanes (consecutive i) touch 256 contiguous bytes per instruction;
    // the upper triangle is mirrored down afterwards (upper_to_lower).
    // All 16 loads are issued before any store (a plain `+=` loop would
    // serialize on possible aliasing between the stores and later loads);
    // 16 columns per step keeps the epilogue inside the converter warps'
    // register budget.
    if (i < q) {
      const int64_t jn = min((int64_t)16, q - (j0 + cc * 16));
      double* col = G + (j0 + cc * 16) * ldg + i;
      double g[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) g[t] = t < jn ? col[t * ldg] : 0.0;
#pragma unroll
      for (int t = 0; t < 16; ++t)
        if (t < jn) col[t * ldg] = fma((double)__uint_as_float(v[t]), unscale, g[t]);
    }
  }
}

template <bool F16>
__global__ void __launch_bounds__(THREADS, 1)
syrk_split_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t K,
                  int64_t q, int64_t kchunk, const int2* __restrict__ tiles, double* __restrict__ G, int64_t ldg,
                  const unsigned* __restrict__ amax_bits) {
  using S = Split<F16>;
  constexpr int NST = S::NST, STAGE = S::STAGE, A_BYTES = S::A_BYTES, B_BYTES = S::B_BYTES;
  constexpr int LBO_A = S::LBO_A, LBO_B = S::LBO_B, KCH = S::KCH;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[NST], empty[NST], accf[2], acce[2], rfull[NRAW], rempty[NRAW];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int2 tile = tiles[blockIdx.x];
  const int64_t i0 = (int64_t)tile.x * TM, j0 = (int64_t)tile.y * TN;
  const int64_t nstages = (K + BK - 1) / BK;
  const int64_t nchunks = (K + kchunk - 1) / kchunk;
  const int64_t SPC = kchunk / BK;   // stages per chunk

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      bar_init(&full[s], NPROD);
      bar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      bar_init(&accf[a], 1);
      bar_init(&acce[a], 4);
    }
    for (int r = 0; r < NRAW; ++r) {
      bar_init(&rfull[r], 1);
      bar_init(&rempty[r], NPROD);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  unsigned char* raw = smem + (size_t)NST * STAGE;
  if (warp == LOADER_WARP) {
    // ===================== TMA loader =====================
    if (lane == 0) {
      for (int64_t it = 0; it < nstages; ++it) {
        const int r = (int)(it % NRAW);
        if (it >= NRAW) bar_wait(&rempty[r], (unsigned)(((it / NRAW) - 1) & 1));
        const int k0 = (int)(it * BK);
        const uint32_t dst = su32(raw + (size_t)r * RAW_BYTES), bar = su32(&rfull[r]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((unsigned)RAW_BYTES)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                dst),
            "l"(&tmA), "r"((int)i0), "r"(k0), "r"(bar)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                dst + RAW_A),
            "l"(&tmB), "r"((int)j0), "r"(k0), "r"(bar)
            : "memory");
      }
    }
  } else if (warp >= 5) {
    // ===================== converters =====================
    // item = (4-row K chunk kc, column c of the A|B panel): 4 conflict-free
    // shared loads down the raw column, split into hi/lo, one 16-byte store of
    // each into the K-major no-swizzle core-matrix layout (consecutive threads
    // -> consecutive columns -> consecutive 16 B rows of a core matrix).
    constexpr int NITEM = ((BK / KCH) * (TM + TN)) / (NPROD * 32);   // 6 (tf32) / 3 (f16)
    const int pt = tid - 5 * 32;   // 0 .. NPROD*32-1
    const float sc = F16 ? ldexpf(1.0f, split_shift(amax_bits)) : 1.0f;
    for (int64_t it = 0; it < nstages; ++it) {
      const int r = (int)(it % NRAW);
      const int s = (int)(it % NST);
      bar_wait(&rfull[r], (unsigned)((it / NRAW) & 1));
      if (it >= NST) bar_wait(&empty[s], (unsigned)(((it / NST) - 1) & 1));
      const float* rs = reinterpret_cast<const float*>(raw + (size_t)r * RAW_BYTES);
      unsigned char* st = smem + (size_t)s * STAGE;
#pragma unroll
      for (int u = 0; u < NITEM; ++u) {
        const int idx = u * NPROD * 32 + pt;
        const int kc = idx / (TM + TN);
        const int c = idx % (TM + TN);
        const bool isA = c < TM;
        const int mn = isA ? c : c - TM;
        const float* col = isA ? rs + mn : rs + BK * TM + mn;
        const int w = isA ? TM : TN;
        float f[KCH];
#pragma unroll
        for (int e = 0; e < KCH; ++e) f[e] = col[(KCH * kc + e) * w];
        uint4 hi, lo;
        if constexpr (F16) {
          uint32_t h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x0 = f[2 * e] * sc, x1 = f[2 * e + 1] * sc;
            h[e] = pack_f16(x0, x1);
            const __half2 hh = *reinterpret_cast<const __half2*>(&h[e]);
            l[e] = pack_f16(x0 - __low2float(hh), x1 - __high2float(hh));
          }
          hi = make_uint4(h[0], h[1], h[2], h[3]);
          lo = make_uint4(l[0], l[1], l[2], l[3]);
        } else {
          hi.x = to_tf32(f[0]); lo.x = to_tf32(f[0] - __uint_as_float(hi.x));
          hi.y = to_tf32(f[1]); lo.y = to_tf32(f[1] - __uint_as_float(hi.y));
          hi.z = to_tf32(f[2]); lo.z = to_tf32(f[2] - __uint_as_float(hi.z));
          hi.w = to_tf32(f[3]); lo.w = to_tf32(f[3] - __uint_as_float(hi.w));
        }
        unsigned char* base_hi = isA ? st : st + 2 * A_BYTES;
        const int lbo = isA ? LBO_A : LBO_B;
        const int nb = isA ? A_BYTES : B_BYTES;
        const int off = kc * lbo + (mn >> 3) * 128 + (mn & 7) * 16;
        *reinterpret_cast<uint4*>(base_hi + off) = hi;
        *reinterpret_cast<uint4*>(base_hi + nb + off) = lo;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        bar_arrive(&full[s]);
        bar_arrive(&rempty[r]);
      }
    }
  } else if (warp == 4) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      for (int64_t c = 0; c < nchunks; ++c) {
        const int acc = (int)(c & 1);
        if (c >= 2) bar_wait(&acce[acc], (unsigned)(((c >> 1) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(acc * TN);
        const int64_t it0 = c * SPC, it1 = min(nstages, it0 + SPC);
        for (int64_t it = it0; it < it1; ++it) {
          const int s = (int)(it % NST);
          bar_wait(&full[s], (unsigned)((it / NST) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t st = su32(smem + (size_t)s * STAGE);
          const uint32_t a_hi = st, a_lo = st + A_BYTES, b_hi = st + 2 * A_BYTES, b_lo = b_hi + B_BYTES;
#pragma unroll
          for (int kk = 0; kk < S::KSTEPS; ++kk) {
            // one MMA covers two K chunks of KCH elements (K = 8 tf32 / 16 f16)
            const uint64_t dah = smem_desc(a_hi + 2 * kk * LBO_A, LBO_A, 128);
            const uint64_t dal = smem_desc(a_lo + 2 * kk * LBO_A, LBO_A, 128);
            const uint64_t dbh = smem_desc(b_hi + 2 * kk * LBO_B, LBO_B, 128);
            const uint64_t dbl = smem_desc(b_lo + 2 * kk * LBO_B, LBO_B, 128);
            const uint32_t accum = (it > it0 || kk > 0) ? 1u : 0u;
            mma_split<F16>(d, dah, dbh, accum);
            mma_split<F16>(d, dah, dbl, 1u);
            mma_split<F16>(d, dal, dbh, 1u);
          }
          mma_commit(&empty[s]);   // frees the stage once these MMAs have read it
        }
        mma_commit(&accf[acc]);    // accumulator ready for the epilogue
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue (warps 0-3) =====================
    const int64_t i = i0 + warp * 32 + lane;   // TMEM lane = tile row
    const double unscale = F16 ? ldexp(1.0, -2 * split_shift(amax_bits)) : 1.0;
    for (int64_t c = 0; c < nchunks; ++c) {
      const int acc = (int)(c & 1);
      bar_wait(&accf[acc], (unsigned)((c >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      drain_chunk(tmem, warp, acc, i, j0, q, G, ldg, unscale);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&acce[acc]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ---- pre-split variant -------------------------------------------------
// The converters above split every panel once per tile that reads it (~20x
// for q = 5000), and their shared-memory traffic is what bounds the kernel.
// When there is room for a second copy of A (4 bytes per element), one
// streaming pass writes hi/lo once, already in the MMA's K-major core-matrix
// order: element (r, c) at [(r / 8) * ncp + c] * 8 + r % 8 (fp16), zero past
// the matrix.  The Gram kernel then only moves bytes: bulk copies straight
// into the operand stages, three MMAs per stage, no conversion warps.
__global__ void __launch_bounds__(256) split_f16_kernel(const float* __restrict__ A, int64_t m, int64_t ld, int64_t n,
                                                        int64_t ncp, int64_t nkb,
                                                        const unsigned* __restrict__ amax_bits,
                                                        uint4* __restrict__ hi, uint4* __restrict__ lo) {
  const float sc = ldexpf(1.0f, split_shift(amax_bits));
  for (int64_t idx = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; idx < nkb * ncp;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kb = idx / ncp, c = idx - kb * ncp;
    float f[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int64_t r = kb * 8 + e;
      f[e] = (r < m && c < n) ? A[r * ld + c] : 0.0f;
    }
    uint32_t h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float x0 = f[2 * e] * sc, x1 = f[2 * e + 1] * sc;
      h[e] = pack_f16(x0, x1);
      const __half2 hh = *reinterpret_cast<const __half2*>(&h[e]);
      l[e] = pack_f16(x0 - __low2float(hh), x1 - __high2float(hh));
    }
    hi[idx] = make_uint4(h[0], h[1], h[2], h[3]);
    lo[idx] = make_uint4(l[0], l[1], l[2], l[3]);
  }
}

// 16-row slabs per stage: the per-stage round trip (copies land -> MMAs ->
// commit -> slot refilled) costs about as much as a slab's MMAs, so stages
// are 4 slabs (96 KB, 12 MMAs) deep and only two are needed: 1 slab per
// stage 16.7 ms, 2 -> 15.0 ms, 4 -> 14.1 ms at 200000 x 5000
constexpr int PRE_SUB = 4;
constexpr int PRE_NST = 8 / PRE_SUB;                        // 192 KB of operand stages
constexpr int PRE_THREADS = 6 * 32;                         // epilogue 0-3, MMA 4, loader 5
constexpr int PRE_SMEM = PRE_NST * PRE_SUB * Split<true>::STAGE;

// CL = 2: a cluster of two CTAs computes tiles (I, J) and (I', J); each
// loads its own A panel and HALF of the shared B panel, multicast into both
// CTAs' stages -- 16 KB of L2 reads per CTA and stage instead of 24 KB (the
// single-CTA kernel runs at the L2->SM bandwidth, ~7.5 TB/s).  Stage s may
// be refilled only when both CTAs' MMAs have read it, so each MMA commit
// arrives on the empty barriers of both CTAs.  A tile with x < 0 is the
// partner of an odd tile count: it loads and multiplies but does not drain.
template <int CL>
__global__ void __launch_bounds__(PRE_THREADS, 1)
syrk_pre_kernel(const unsigned char* __restrict__ hi, const unsigned char* __restrict__ lo, int64_t ncp, int64_t nkb,
                int64_t q, int64_t kchunk, const int2* __restrict__ tiles, double* __restrict__ G, int64_t ldg,
                const unsigned* __restrict__ amax_bits) {
  using S = Split<true>;
  constexpr int STAGE = S::STAGE, A_BYTES = S::A_BYTES, B_BYTES = S::B_BYTES, LBO_A = S::LBO_A, LBO_B = S::LBO_B;
  constexpr int BW = TN / CL;                                // B columns this CTA loads
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[PRE_NST], empty[PRE_NST], accf[2], acce[2];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int2 tile = tiles[blockIdx.x];
  const bool drain = tile.x >= 0;
  const int64_t i0 = (int64_t)(drain ? tile.x : -tile.x - 1) * TM, j0 = (int64_t)tile.y * TN;
  uint32_t rank = 0;
  if constexpr (CL > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int64_t nstages = nkb / (2 * PRE_SUB);              // 16 PRE_SUB rows per stage
  const int64_t nchunks = (nstages * BK * PRE_SUB + kchunk - 1) / kchunk;
  const int64_t SPC = kchunk / (BK * PRE_SUB);

  if (tid == 0) {
    for (int s = 0; s < PRE_NST; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], CL);
    }
    for (int a = 0; a < 2; ++a) {
      bar_init(&accf[a], 1);
      bar_init(&acce[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (CL > 1) {   // peers' barriers are initialised before anyone multicasts into them
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  if (warp == 5) {
    // ===================== loader =====================
    if (lane == 0) {
      const int64_t row_bytes = ncp * 16;                   // one 8-row block, all columns
      const uint16_t mask = (uint16_t)((1u << CL) - 1u);
      for (int64_t it = 0; it < nstages; ++it) {
        const int s = (int)(it % PRE_NST);
        if (it >= PRE_NST) bar_wait(&empty[s], (unsigned)(((it / PRE_NST) - 1) & 1));
        const uint32_t st0 = su32(smem + (size_t)s * PRE_SUB * STAGE), bar = su32(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((unsigned)(PRE_SUB * STAGE))
                     : "memory");
#pragma unroll
        for (int sub = 0; sub < PRE_SUB; ++sub)
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          const int64_t kb = 2 * (it * PRE_SUB + sub) + kc;
          const uint32_t st = st0 + sub * STAGE;
          const unsigned char* srcs[2] = {hi, lo};
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const unsigned char* base = srcs[part] + kb * row_bytes;
            const uint32_t da = st + part * A_BYTES + kc * LBO_A;
            const uint32_t db = st + 2 * A_BYTES + part * B_BYTES + kc * LBO_B + rank * (BW * 16);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(da),
                "l"(base + i0 * 16), "r"((unsigned)(TM * 16)), "r"(bar)
                : "memory");
            if constexpr (CL > 1)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, "
                  "[%3], %4;" ::"r"(db),
                  "l"(base + (j0 + rank * BW) * 16), "r"((unsigned)(BW * 16)), "r"(bar), "h"(mask)
                  : "memory");
            else
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(db),
                  "l"(base + j0 * 16), "r"((unsigned)(TN * 16)), "r"(bar)
                  : "memory");
          }
        }
      }
    }
  } else if (warp == 4) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      for (int64_t c = 0; c < nchunks; ++c) {
        const int acc = (int)(c & 1);
        if (c >= 2) bar_wait(&acce[acc], (unsigned)(((c >> 1) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(acc * TN);
        const int64_t it0 = c * SPC, it1 = min(nstages, it0 + SPC);
        for (int64_t it = it0; it < it1; ++it) {
          const int s = (int)(it % PRE_NST);
          bar_wait(&full[s], (unsigned)((it / PRE_NST) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int sub = 0; sub < PRE_SUB; ++sub) {
            const uint32_t st = su32(smem + ((size_t)s * PRE_SUB + sub) * STAGE);
            const uint32_t a_hi = st, a_lo = st + A_BYTES, b_hi = st + 2 * A_BYTES, b_lo = b_hi + B_BYTES;
            const uint64_t dah = smem_desc(a_hi, LBO_A, 128), dal = smem_desc(a_lo, LBO_A, 128);
            const uint64_t dbh = smem_desc(b_hi, LBO_B, 128), dbl = smem_desc(b_lo, LBO_B, 128);
            mma_split<true>(d, dah, dbh, (it > it0 || sub > 0) ? 1u : 0u);
            mma_split<true>(d, dah, dbl, 1u);
            mma_split<true>(d, dal, dbh, 1u);
          }
          if constexpr (CL > 1)
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    su32(&empty[s])),
                "h"((uint16_t)((1u << CL) - 1u))
                : "memory");
          else
            mma_commit(&empty[s]);
        }
        mma_commit(&accf[acc]);
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue (warps 0-3) =====================
    const int64_t i = i0 + warp * 32 + lane;
    const double unscale = ldexp(1.0, -2 * split_shift(amax_bits));
    for (int64_t c = 0; c < nchunks; ++c) {
      const int acc = (int)(c & 1);
      bar_wait(&accf[acc], (unsigned)((c >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (drain) drain_chunk(tmem, warp, acc, i, j0, q, G, ldg, unscale);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&acce[acc]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (CL > 1) {   // no CTA leaves while its peer may still write or arrive into its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ---- fp64 Gram on the int8 tensor cores -------------------------------
// G = A'A for fp64 A (tall) without the fp64 pipe: every column c is scaled
// by 2^-e_c (e_c: exponent of max_i |A_ic|, exact) into (-1, 1) and cut into
// I8_S = 8 signed slices by round-to-nearest,
//     x = q_1 2^-6 + q_2 2^-13 + ... + q_8 2^-55 + r,   q_s in [-64, 64],
// |r| <= 2^-56 (every step exact in fp64; the signed remainders keep the
// dropped terms unbiased -- truncated slices all share x's sign and biased
// the diagonal by ~1e-13).  Products of int8 slices accumulate EXACTLY in
// int32 on the tensor cores (kind::i8), so
//     (A'A)_jk = 2^(e_j + e_k) sum_{s+t <= S+1} 2^(2 - 7 (s+t)) (Q_s' Q_t)_jk
// is exact up to the slicing remainder and the dropped pairs s + t >= S + 2
// (~2^-56 of max|A_j| max|A_k| per row, unbiased): at or below the rounding
// of an fp64 dot product (the Ozaki scheme with integer slices; the error is
// "fixed point" relative to the column maxima -- seven slices left ~1e-14
// absolute on O(1) entries).  One int32 TMEM accumulator per anti-diagonal
// d = s + t (the pairs on it share the weight): S accumulators of 64
// columns = all 512 TMEM columns, drained into the fp64 G every I8_KCHUNK
// rows (int32 bound: S * 64^2 * rows < 2^31).
//
// Slices live in the MMA's K-major core-matrix order, slice-major:
// byte (s, r, c) at s * slice_bytes + ((r / 16) * ncp + c) * 16 + r % 16.  A
// 4-D tensor map (a panel's 16-byte K rows as one run, column blocks, 16-row
// blocks, slices) moves a stage -- I8_NK 16-row blocks of every slice of the
// 128-column A panel, and of the 64-column B panel -- in ONE copy each,
// straight into the layout the descriptors read (A: K-block stride 2 KB,
// B: 1 KB; 8-row groups 128 B apart).  Warp roles as in syrk_pre_kernel:
// epilogue 0-3, MMA 4, loader 5.
constexpr int I8_S = 8;                        // slices (7 bits each; anti-diagonals kept: S)
constexpr int I8_TN = 64;                      // tile columns: I8_S x 64 TMEM columns <= 512
constexpr int I8_NK = 4;                       // 16-row K blocks per stage (2 MMAs of K = 32)
constexpr int I8_NST = 2;                      // stages
constexpr int I8_KCHUNK = 32768;               // rows per int32 accumulation
constexpr int I8_A_SLICE = I8_NK * TM * 16;    // 8 KB
constexpr int I8_B_SLICE = I8_NK * I8_TN * 16; // 4 KB
constexpr int I8_A_STAGE = I8_S * I8_A_SLICE;  // 64 KB
constexpr int I8_STAGE = I8_S * (I8_A_SLICE + I8_B_SLICE);   // 96 KB
constexpr int I8_SMEM = I8_NST * I8_STAGE;     // 192 KB
constexpr int I8_THREADS = 6 * 32;
// D s32 (2), A/B signed int8 (1), K-major, N = 64, M = 128
constexpr uint32_t I8_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(I8_TN >> 3) << 17) |
                              ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(I8_IDESC), "r"(accumulate));
}

// per-column max |A| as fp64 bits (non-negative doubles order like their bits)
__global__ void colmax_f64_kernel(const double* __restrict__ A, int64_t m, int64_t ld, int64_t n,
                                  unsigned long long* __restrict__ cmax) {
  const int64_t rows_per = (m + gridDim.y - 1) / gridDim.y;
  const int64_t r0 = blockIdx.y * rows_per, r1 = min(m, r0 + rows_per);
  for (int64_t c = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    double mx = 0.0;
    for (int64_t r = r0; r < r1; ++r) mx = fmax(mx, fabs(A[r * ld + c]));
    if (mx > 0.0) atomicMax(cmax + c, (unsigned long long)__double_as_longlong(mx));
  }
}

// slices of the 16-row block kb, column c (one thread each): 16 doubles in,
// I8_S x 16 int8 out (one 16-byte store per slice)
__global__ void __launch_bounds__(256) slice_i8_kernel(const double* __restrict__ A, int64_t m, int64_t ld, int64_t n,
                                                       int64_t ncp, int64_t nkb,
                                                       const unsigned long long* __restrict__ cmax,
                                                       uint4* __restrict__ Q, int64_t slice_vecs) {
  for (int64_t idx = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; idx < nkb * ncp;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kb = idx / ncp, c = idx - kb * ncp;
    int e = 0;
    if (c < n) {
      const double mx = __longlong_as_double((long long)cmax[c]);
      if (mx > 0.0) frexp(mx, &e);   // mx in [2^(e-1), 2^e)
    }
    double r[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int64_t row = kb * 16 + t;
      r[t] = (row < m && c < n) ? ldexp(A[row * ld + c], 6 - e) : 0.0;   // (-64, 64)
    }
#pragma unroll
    for (int sl = 0; sl < I8_S; ++sl) {
      uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const double qd = rint(r[t]);             // |qd| <= 64
        r[t] = (r[t] - qd) * 128.0;               // exact, [-64, 64]
        w[t >> 2] |= ((uint32_t)(int)qd & 0xffu) << (8 * (t & 3));
      }
      Q[sl * slice_vecs + idx] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

__global__ void colexp_kernel(const unsigned long long* __restrict__ cmax, int64_t n, int* __restrict__ ex) {
  for (int64_t c = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    int e = 0;
    const double mx = __longlong_as_double((long long)cmax[c]);
    if (mx > 0.0) frexp(mx, &e);
    ex[c] = e;
  }
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}

__global__ void __launch_bounds__(I8_THREADS, 1)
syrk_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t nkb,
               int64_t q, const int2* __restrict__ tiles, const int* __restrict__ ex, double* __restrict__ G,
               int64_t ldg) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[I8_NST], empty[I8_NST], accf, acce;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int2 tile = tiles[blockIdx.x];
  const int64_t i0 = (int64_t)tile.x * TM, j0 = (int64_t)tile.y * I8_TN;
  const int64_t nstages = nkb / I8_NK;
  const int64_t SPC = I8_KCHUNK / (16 * I8_NK);
  const int64_t nchunks = (nstages + SPC - 1) / SPC;

  if (tid == 0) {
    for (int s = 0; s < I8_NST; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], 1);
    }
    bar_init(&accf, 1);
    bar_init(&acce, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  if (warp == 5) {
    // ===================== loader: two tensor copies per stage =====================
    if (lane == 0) {
      for (int64_t it = 0; it < nstages; ++it) {
        const int s = (int)(it % I8_NST);
        if (it >= I8_NST) bar_wait(&empty[s], (unsigned)(((it / I8_NST) - 1) & 1));
        const uint32_t st = su32(smem + (size_t)s * I8_STAGE), bar = su32(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((unsigned)I8_STAGE)
                     : "memory");
        const int kb = (int)(it * I8_NK);
        tma_load_4d(st, &tmA, 0, (int)(i0 / TM), kb, 0, bar);
        tma_load_4d(st + I8_A_STAGE, &tmB, 0, (int)(j0 / I8_TN), kb, 0, bar);
      }
    }
  } else if (warp == 4) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t LBO_A = TM * 16, LBO_B = I8_TN * 16;
      for (int64_t c = 0; c < nchunks; ++c) {
        if (c >= 1) bar_wait(&acce, (unsigned)((c - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int64_t it0 = c * SPC, it1 = min(nstages, it0 + SPC);
        for (int64_t it = it0; it < it1; ++it) {
          const int s = (int)(it % I8_NST);
          bar_wait(&full[s], (unsigned)((it / I8_NST) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = su32(smem + (size_t)s * I8_STAGE), sb = sa + I8_A_STAGE;
#pragma unroll
          for (int kk = 0; kk < I8_NK / 2; ++kk) {
#pragma unroll
            for (int ps = 0; ps < I8_S; ++ps)
#pragma unroll
              for (int pt = 0; pt + ps < I8_S; ++pt) {   // s + t <= S + 1 with 1-based slices
                const uint64_t da = smem_desc(sa + ps * I8_A_SLICE + 2 * kk * LBO_A, LBO_A, 128);
                const uint64_t db = smem_desc(sb + pt * I8_B_SLICE + 2 * kk * LBO_B, LBO_B, 128);
                const int d = ps + pt;                   // anti-diagonal: accumulator d
                // the first product into each accumulator of a chunk overwrites it
                mma_i8(tmem + (uint32_t)(d * I8_TN), da, db, (it > it0 || kk > 0 || ps > 0) ? 1u : 0u);
              }
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&accf);
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue (warps 0-3): drain into fp64 G =====================
    const int64_t i = i0 + warp * 32 + lane;
    const int ei = i < q ? ex[i] : 0;
    for (int64_t c = 0; c < nchunks; ++c) {
      bar_wait(&accf, (unsigned)(c & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int cc = 0; cc < I8_TN / 16; ++cc) {
        uint32_t v[I8_S][16];
#pragma unroll
        for (int d = 0; d < I8_S; ++d) {
          const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(d * I8_TN + cc * 16);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
              "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[d][0]), "=r"(v[d][1]), "=r"(v[d][2]), "=r"(v[d][3]), "=r"(v[d][4]), "=r"(v[d][5]),
                "=r"(v[d][6]), "=r"(v[d][7]), "=r"(v[d][8]), "=r"(v[d][9]), "=r"(v[d][10]), "=r"(v[d][11]),
                "=r"(v[d][12]), "=r"(v[d][13]), "=r"(v[d][14]), "=r"(v[d][15])
              : "r"(taddr));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (i < q) {
          const int64_t jb = j0 + cc * 16;
          const int64_t jn = min((int64_t)16, q - jb);
          double* col = G + jb * ldg + i;
          double g[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) g[t] = t < jn ? col[t * ldg] : 0.0;
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            if (t >= jn) continue;
            // Horner from the least significant anti-diagonal: sum_d 2^(-7 d - 12) acc_d
            double sum = (double)(int)v[I8_S - 1][t];
#pragma unroll
            for (int d = I8_S - 2; d >= 0; --d) sum = fma(sum, 0x1p-7, (double)(int)v[d][t]);
            col[t * ldg] = g[t] + ldexp(sum, ei + ex[jb + t] - 12);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&acce);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ---- pre-split Gram on CTA pairs (tcgen05 cta_group::2; opt-in) -----------
// The 2-CTA cluster above shares the B panel by multicast, but each SM still
// takes 24 KB of operands into shared memory per 16-row slab for 128 x 256
// MACs (ncu: 14.3 ms against a 9 ms f16 floor at 200000 x 5000).  Here the
// two SMs run ONE 256 x 256
// MMA (cta_group::2): CTA r holds rows [128 r, 128 r + 128) of the A panel
// (its TMEM lanes: its half of the tile) and columns [128 r, 128 r + 128) of
// the B panel, 16 KB per slab per SM for the same MACs per SM.  The leader
// (rank 0) issues the MMAs; both CTAs' tensor copies (cta_group::2) complete
// on the leader's `full` barrier; MMA commits are multicast to both CTAs'
// `empty` / `accf`; each CTA drains its own TMEM half into G and its epilogue
// warps arrive on the leader's `acce` (count 8).  A stage is four slabs of
// hi and lo for A and B: one 4-D copy (16-byte K rows of a 128-column panel,
// column block, 8-row block, hi/lo) per operand.
constexpr int P2_STAGE = 4 * PRE_SUB * 128 * 16 * 2;      // (A, B) x (hi, lo) x 4 slabs x 2 KB = 64 KB
constexpr int P2_NST = 3;
constexpr int P2_SMEM = P2_NST * P2_STAGE;                 // 192 KB
constexpr uint32_t P2_IDESC = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(256 >> 3) << 17) |
                              ((uint32_t)(256 >> 4) << 24);   // D f32, A/B f16, K-major, N = 256, M = 256

__device__ __forceinline__ void tma4_cg2(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                         uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5}], [%6];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(leader_bar)
      : "memory");
}

__global__ void __launch_bounds__(PRE_THREADS, 1)
syrk_pre2sm_kernel(const __grid_constant__ CUtensorMap tm, int64_t nkb, int64_t q, int64_t kchunk,
                   const int2* __restrict__ tiles, double* __restrict__ G, int64_t ldg,
                   const unsigned* __restrict__ amax_bits) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[P2_NST], empty[P2_NST], accf[2], acce[2];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const bool leader = rank == 0;
  const int2 tile = tiles[blockIdx.x >> 1];
  const int64_t I0 = (int64_t)tile.x * 256, j0 = (int64_t)tile.y * 256;
  const int64_t i0 = I0 + 128 * rank;                          // this CTA's A rows = TMEM lanes
  const int64_t nstages = nkb / (2 * PRE_SUB);                 // 8 eight-row blocks (64 rows) per stage
  const int64_t SPC = kchunk / (BK * PRE_SUB);
  const int64_t nchunks = (nstages + SPC - 1) / SPC;

  if (tid == 0) {
    for (int s = 0; s < P2_NST; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      bar_init(&accf[a], 1);
      bar_init(&acce[a], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;
  const uint32_t peer_mask = 0xFEFFFFFFu;                      // shared::cluster address -> the leader's copy

  if (warp == 5) {
    // ===================== loader (both CTAs) =====================
    if (lane == 0) {
      for (int64_t it = 0; it < nstages; ++it) {
        const int s = (int)(it % P2_NST);
        if (it >= P2_NST) bar_wait(&empty[s], (unsigned)(((it / P2_NST) - 1) & 1));
        const uint32_t st = su32(smem + (size_t)s * P2_STAGE);
        const uint32_t bar = su32(&full[s]) & peer_mask;
        if (leader)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                       "r"((unsigned)(2 * P2_STAGE))
                       : "memory");
        const int kb = (int)(it * 2 * PRE_SUB);
        tma4_cg2(st, &tm, 0, (int)(i0 / 128), kb, 0, bar);                              // A rows: hi, lo
        tma4_cg2(st + P2_STAGE / 2, &tm, 0, (int)(j0 / 128) + (int)rank, kb, 0, bar);     // B half: hi, lo
      }
    }
  } else if (warp == 4) {
    // ===================== MMA issuer (leader) =====================
    if (leader && lane == 0) {
      constexpr uint32_t SL = 2 * PRE_SUB * 128 * 16;          // one operand part (hi or lo): 8 blocks x 2 KB
      constexpr uint32_t LBO = 128 * 16;                       // next 8-row block
      for (int64_t c = 0; c < nchunks; ++c) {
        const int acc = (int)(c & 1);
        if (c >= 2) bar_wait(&acce[acc], (unsigned)(((c >> 1) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(acc * TN);
        const int64_t it0 = c * SPC, it1 = min(nstages, it0 + SPC);
        for (int64_t it = it0; it < it1; ++it) {
          const int s = (int)(it % P2_NST);
          bar_wait(&full[s], (unsigned)((it / P2_NST) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a_hi = su32(smem + (size_t)s * P2_STAGE), a_lo = a_hi + SL;
          const uint32_t b_hi = a_hi + P2_STAGE / 2, b_lo = b_hi + SL;
#pragma unroll
          for (int sub = 0; sub < PRE_SUB; ++sub) {            // K = 16: two 8-row blocks per MMA
            const uint32_t off = (uint32_t)(2 * sub) * LBO;
            const uint64_t dah = smem_desc(a_hi + off, LBO, 128), dal = smem_desc(a_lo + off, LBO, 128);
            const uint64_t dbh = smem_desc(b_hi + off, LBO, 128), dbl = smem_desc(b_lo + off, LBO, 128);
            const uint32_t accum = (it > it0 || sub > 0) ? 1u : 0u;
#pragma unroll
            for (int pr = 0; pr < 3; ++pr) {
              const uint64_t da = pr == 2 ? dal : dah, db = pr == 1 ? dbl : dbh;
              asm volatile(
                  "{\n\t.reg .pred p;\n\t"
                  "setp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                  "l"(da), "l"(db), "r"(P2_IDESC), "r"(pr == 0 ? accum : 1u));
            }
          }
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  su32(&empty[s])),
              "h"((uint16_t)3)
              : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                su32(&accf[acc])),
            "h"((uint16_t)3)
            : "memory");
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ===================== epilogue (warps 0-3, both CTAs) =====================
    const int64_t i = i0 + warp * 32 + lane;
    const double unscale = ldexp(1.0, -2 * split_shift(amax_bits));
    for (int64_t c = 0; c < nchunks; ++c) {
      const int acc = (int)(c & 1);
      bar_wait(&accf[acc], (unsigned)((c >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      drain_chunk(tmem, warp, acc, i, j0, q, G, ldg, unscale);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {   // the leader's acce: local arrive, or a remote one from the peer
        if (leader) {
          bar_arrive(&acce[acc]);
        } else {
          const uint32_t rb = su32(&acce[acc]) & peer_mask;
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// The kernel accumulates the upper triangle (transposed tile writes); copy it
// down so callers see the usual lower-triangle result.
__global__ void upper_to_lower(double* G, int64_t q, int64_t ld) {
  const int64_t i = blockIdx.y * (int64_t)blockDim.y + threadIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < q && j < i) G[i * ld + j] = G[j * ld + i];
}

}  // namespace syrk

// 2-D tensor map over the fp32 matrix (ld columns x m rows, row stride ld*4)
// with a BK x box_cols box, no swizzle, zero fill out of bounds.  The driver
// entry point comes through the runtime (no libcuda link dependency).
static CUtensorMap panel_map(const gf_matrix* A, int box_cols) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    GF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    GF_REQUIRE(fn != nullptr && q == cudaDriverEntryPointSuccess, GF_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)A->ld, (cuuint64_t)A->m};
  const cuuint64_t strides[1] = {(cuuint64_t)A->ld * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)syrk::BK};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A->data, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  GF_REQUIRE(r == CUDA_SUCCESS, GF_E_CUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

static bool gram_i8_enabled() {
  const char* e = getenv("GF_GRAM_F64");   // "dmma": the fp64 tensor-core GEMM instead of the int8 slices
  return !(e && std::string(e) == "dmma");
}

static int64_t i8_ncp(int64_t q) { return ceil_div(q, syrk::TM) * syrk::TM; }
static int64_t i8_nkb(int64_t m) { return ceil_div(m, 16 * syrk::I8_NK) * syrk::I8_NK; }

size_t gram_scratch_bytes(const gf_matrix* A, bool tall) {
  if (tall && A->dtype == GF_F64)
    return gram_i8_enabled() ? (size_t)syrk::I8_S * i8_nkb(A->m) * i8_ncp(A->n) * 16 : 0;
  const char* sp = getenv("GF_SYRK");   // "tf32" / "f16": the in-kernel converters, no copy
  if (!tall || A->dtype != GF_F32 || (sp && (std::string(sp) == "tf32" || std::string(sp) == "f16"))) return 0;
  const int64_t ncp = ceil_div(A->n, syrk::TN) * syrk::TN, nkb = ceil_div(A->m, syrk::BK * syrk::PRE_SUB) * 2 * syrk::PRE_SUB;
  return 2 * (size_t)nkb * ncp * 16;
}

// max |A| over the n real columns, as float bits (non-negative floats order
// like their bit patterns); the padding columns are not read
__global__ void absmax_kernel(const float* __restrict__ A, int64_t m, int64_t ld, int64_t n,
                              unsigned* __restrict__ out) {
  const int nv = (int)((n + 3) / 4);
  float mx = 0.0f;
  for (int64_t r = blockIdx.x; r < m; r += gridDim.x) {
    const float4* row = reinterpret_cast<const float4*>(A + r * ld);
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
      const float4 a = row[v];
      const int j = 4 * v;
      mx = fmaxf(mx, fabsf(a.x));
      if (j + 1 < n) mx = fmaxf(mx, fabsf(a.y));
      if (j + 2 < n) mx = fmaxf(mx, fabsf(a.z));
      if (j + 3 < n) mx = fmaxf(mx, fabsf(a.w));
    }
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(mx));
}

// G (fp64, zeroed by the caller) += A'A for fp32 A (m x ld, columns >= n zero).
// Default split: scaled fp16 hi/lo (kind::f16); GF_SYRK=tf32 selects 3xTF32.
void gram_tf32x3(const gf_matrix* A, double* G, int64_t ldg, cudaStream_t st, void* scratch, size_t scratch_bytes,
                 const unsigned* amax_known) {
  using namespace syrk;
  const int64_t q = A->n;
  const int64_t bi_n = ceil_div(q, TM), bj_n = ceil_div(q, TN);
  std::vector<int2> tl;
  for (int64_t bi = 0; bi < bi_n; ++bi)
    for (int64_t bj = 0; bj < bj_n; ++bj)
      if (2 * bj <= bi) tl.push_back(make_int2((int)bi, (int)bj));   // lower-triangle tiles
  DBuf d_tiles(tl.size() * sizeof(int2) + 16);
  GF_CUDA(cudaMemcpyAsync(d_tiles.p, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  const char* sp = getenv("GF_SYRK");
  const bool f16 = !(sp && std::string(sp) == "tf32");
  const int64_t ncp = ceil_div(q, TN) * TN, nkb = ceil_div(A->m, BK * PRE_SUB) * 2 * PRE_SUB;
  const size_t pre_bytes = (size_t)nkb * ncp * 16;          // each of hi, lo
  const bool pre = f16 && scratch != nullptr && scratch_bytes >= 2 * pre_bytes;
  static bool attr[2] = {false, false};
  if (!attr[f16]) {
    if (f16)
      GF_CUDA(cudaFuncSetAttribute(syrk_split_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   Split<true>::SMEM));
    else
      GF_CUDA(cudaFuncSetAttribute(syrk_split_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   Split<false>::SMEM));
    attr[f16] = true;
  }
  const char* kc_env = getenv("GF_SYRK_KCHUNK");
  int64_t kchunk = kc_env ? std::max<int64_t>(BK, atoll(kc_env) / BK * BK) : KCHUNK_DEFAULT;
  const CUtensorMap tmA = panel_map(A, TM), tmB = panel_map(A, TN);
  unsigned* amax = reinterpret_cast<unsigned*>(d_tiles.as<char>() + tl.size() * sizeof(int2) + 8);
  if (f16) {
    if (amax_known != nullptr) {   // max |A_hat| from the scaling pass
      GF_CUDA(cudaMemcpyAsync(amax, amax_known, sizeof(unsigned), cudaMemcpyDeviceToDevice, st));
    } else {
      GF_CUDA(cudaMemsetAsync(amax, 0, sizeof(unsigned), st));
      absmax_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(A->m, num_sms() * 8)), 256, 0, st>>>(
          (const float*)A->data, A->m, A->ld, q, amax);
      GF_CHECK_LAUNCH();
    }
    if (pre) {
      // cluster pairs share a B panel: per column block bj the tiles bi are
      // paired in order; an odd count gets a non-draining partner
      const char* ce = getenv("GF_SYRK_CLUSTER");
      const bool cl2 = !(ce && ce[0] == '1');
      std::vector<int2> tl2;
      for (int64_t bj = 0; bj < bj_n; ++bj) {
        int cnt = 0;
        for (int64_t bi = 2 * bj; bi < bi_n; ++bi, ++cnt) tl2.push_back(make_int2((int)bi, (int)bj));
        if (cnt & 1) tl2.push_back(make_int2((int)(-(bi_n - 1) - 1), (int)bj));
      }
      DBuf d_tiles2(cl2 ? tl2.size() * sizeof(int2) : 0);
      if (cl2)
        GF_CUDA(cudaMemcpyAsync(d_tiles2.p, tl2.data(), tl2.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
      static bool pre_attr = false;
      if (!pre_attr) {
        GF_CUDA(cudaFuncSetAttribute(syrk_pre_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, PRE_SMEM));
        GF_CUDA(cudaFuncSetAttribute(syrk_pre_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, PRE_SMEM));
        pre_attr = true;
      }
      const char* vb = getenv("GF_VERBOSE_SETUP");
      const bool verbose = vb && vb[0] == '1';
      cudaEvent_t ev[3];
      if (verbose)
        for (auto& e : ev) GF_CUDA(cudaEventCreate(&e));
      unsigned char* hi = (unsigned char*)scratch;
      unsigned char* lo = hi + pre_bytes;
      if (verbose) GF_CUDA(cudaEventRecord(ev[0], st));
      split_f16_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nkb * ncp, 256), num_sms() * 16), 256, 0, st>>>(
          (const float*)A->data, A->m, A->ld, q, ncp, nkb, amax, (uint4*)hi, (uint4*)lo);
      GF_CHECK_LAUNCH();
      if (verbose) GF_CUDA(cudaEventRecord(ev[1], st));
      // GF_SYRK_2SM=1: the cta_group::2 kernel (correct -- the Gram tests pass
      // on it -- but 18.0 ms against 14.4 ms for the multicast pairs: its
      // operand reads miss L2 three times as often, 32 GB from DRAM per Gram
      // against 11 GB, ncu profiles/r02/ncu_syrk_pre2sm.txt)
      const char* e2 = getenv("GF_SYRK_2SM");
      const bool two_sm = cl2 && (e2 && e2[0] == '1');
      if (two_sm) {
        // 4-D map of the pre-split hi/lo copy (8-byte words): (the 16-byte K rows of
        // a 128-column block, column block, 8-row block, hi/lo)
        static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        if (!encode) {
          cudaDriverEntryPointQueryResult qr;
          void* fn = nullptr;
          GF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
          GF_REQUIRE(fn != nullptr && qr == cudaDriverEntryPointSuccess, GF_E_CUDA, "cuTensorMapEncodeTiled unavailable");
          encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
        }
        const cuuint64_t dims[4] = {256, (cuuint64_t)(ncp / 128), (cuuint64_t)nkb, 2};
        const cuuint64_t strides[3] = {128 * 16, (cuuint64_t)ncp * 16, (cuuint64_t)pre_bytes};
        const cuuint32_t box[4] = {256, 1, (cuuint32_t)(2 * PRE_SUB), 2};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        CUtensorMap tm;
        const CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, scratch, dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        GF_REQUIRE(r == CUDA_SUCCESS, GF_E_CUDA, "cuTensorMapEncodeTiled (fp16 split) failed");
        // 256 x 256 tiles (I2, J), J <= I2, column-block major: the pairs in
        // flight share a B panel (L2 hits; row-major order re-read operands
        // from DRAM, 37.7 GB per Gram at 200000 x 5000)
        std::vector<int2> tp;
        const int64_t nb2 = ceil_div(q, (int64_t)256);
        for (int64_t bj = 0; bj < nb2; ++bj)
          for (int64_t bi = bj; bi < nb2; ++bi) tp.push_back(make_int2((int)bi, (int)bj));
        DBuf d_tp(tp.size() * sizeof(int2));
        GF_CUDA(cudaMemcpyAsync(d_tp.p, tp.data(), tp.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
        static bool attr2 = false;
        if (!attr2) {
          GF_CUDA(cudaFuncSetAttribute(syrk_pre2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, P2_SMEM));
          attr2 = true;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(2 * tp.size()));
        cfg.blockDim = dim3(PRE_THREADS);
        cfg.dynamicSmemBytes = P2_SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        GF_CUDA(cudaLaunchKernelEx(&cfg, syrk_pre2sm_kernel, tm, nkb, q, kchunk, (const int2*)d_tp.as<int2>(), G, ldg,
                                   (const unsigned*)amax));
        GF_CHECK_LAUNCH();
        GF_CUDA(cudaStreamSynchronize(st));   // d_tp is freed on return
      } else if (cl2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)tl2.size());
        cfg.blockDim = dim3(PRE_THREADS);
        cfg.dynamicSmemBytes = PRE_SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        GF_CUDA(cudaLaunchKernelEx(&cfg, syrk_pre_kernel<2>, (const unsigned char*)hi, (const unsigned char*)lo, ncp,
                                   nkb, q, kchunk, (const int2*)d_tiles2.as<int2>(), G, ldg, (const unsigned*)amax));
      } else {
        syrk_pre_kernel<1><<<(unsigned)tl.size(), PRE_THREADS, PRE_SMEM, st>>>(hi, lo, ncp, nkb, q, kchunk,
                                                                           d_tiles.as<int2>(), G, ldg, amax);
      }
      GF_CHECK_LAUNCH();
      if (verbose) GF_CUDA(cudaEventRecord(ev[2], st));
      if (verbose) {
        GF_CUDA(cudaStreamSynchronize(st));
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, ev[0], ev[1]);
        cudaEventElapsedTime(&b, ev[1], ev[2]);
        fprintf(stderr, "[gf] gram pre-split: split %.2f ms, syrk %.2f ms\n", a, b);
        for (auto& e : ev) cudaEventDestroy(e);
      }
    } else {
      syrk_split_kernel<true><<<(unsigned)tl.size(), THREADS, Split<true>::SMEM, st>>>(
          tmA, tmB, A->m, q, kchunk, d_tiles.as<int2>(), G, ldg, amax);
    }
  } else {
    syrk_split_kernel<false><<<(unsigned)tl.size(), THREADS, Split<false>::SMEM, st>>>(
        tmA, tmB, A->m, q, kchunk, d_tiles.as<int2>(), G, ldg, nullptr);
  }
  GF_CHECK_LAUNCH();
  upper_to_lower<<<dim3((unsigned)ceil_div(q, 32), (unsigned)ceil_div(q, 8)), dim3(32, 8), 0, st>>>(G, q, ldg);
  GF_CHECK_LAUNCH();
  GF_CUDA(cudaStreamSynchronize(st));
}

// fp64 tall Gram on the int8 tensor cores (see syrk_i8_kernel); `scratch`
// holds the slices (gram_scratch_bytes).  G (zeroed by the caller) += A'A.
bool gram_f64_i8(const gf_matrix* A, double* G, int64_t ldg, cudaStream_t st, void* scratch, size_t scratch_bytes) {
  using namespace syrk;
  const int64_t m = A->m, q = A->n;
  const int64_t ncp = i8_ncp(q), nkb = i8_nkb(m);
  const size_t slice_bytes = (size_t)nkb * ncp * 16;
  if (!gram_i8_enabled() || scratch == nullptr || scratch_bytes < (size_t)I8_S * slice_bytes || m <= 0 || q <= 0)
    return false;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    GF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
    GF_REQUIRE(fn != nullptr && qr == cudaDriverEntryPointSuccess, GF_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  // 8-byte words: (the 16-byte K rows of a panel's columns -- one contiguous
  // run per 16-row block: 2 KB for the 128 A columns, 1 KB for the 64 B
  // columns --, column blocks, 16-row blocks, slices).  Long inner runs: a
  // 16-byte inner box dimension ran the copy engine at ~16 B per cycle.
  CUtensorMap tmA, tmB;
  for (int w = 0; w < 2; ++w) {
    const int64_t cols = w == 0 ? TM : I8_TN;
    const cuuint64_t dims[4] = {(cuuint64_t)(cols * 2), (cuuint64_t)(ncp / cols), (cuuint64_t)nkb, (cuuint64_t)I8_S};
    const cuuint64_t strides[3] = {(cuuint64_t)cols * 16, (cuuint64_t)ncp * 16, (cuuint64_t)slice_bytes};
    const cuuint32_t box[4] = {(cuuint32_t)(cols * 2), 1, (cuuint32_t)I8_NK, (cuuint32_t)I8_S};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode(w == 0 ? &tmA : &tmB, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, scratch, dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    GF_REQUIRE(r == CUDA_SUCCESS, GF_E_CUDA, "cuTensorMapEncodeTiled (int8 slices) failed");
  }
  std::vector<int2> tl;   // tiles (I: 128 rows of A'A, J: 64 columns) with j0 < i0 + 128: covers j <= i
  for (int64_t bi = 0; bi < ceil_div(q, TM); ++bi)
    for (int64_t bj = 0; bj * I8_TN < std::min((bi + 1) * TM, q); ++bj) tl.push_back(make_int2((int)bi, (int)bj));
  DBuf small(tl.size() * sizeof(int2) + (size_t)q * (sizeof(unsigned long long) + sizeof(int)) + 64);
  int2* d_tiles = small.as<int2>();
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(small.as<char>() + ((tl.size() * sizeof(int2) + 15) / 16) * 16);
  int* ex = reinterpret_cast<int*>(cmax + q);
  GF_CUDA(cudaMemcpyAsync(d_tiles, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  GF_CUDA(cudaMemsetAsync(cmax, 0, q * sizeof(unsigned long long), st));
  const char* vb = getenv("GF_VERBOSE_SETUP");
  const bool verbose = vb && vb[0] == '1';
  cudaEvent_t ev[3];
  if (verbose) {
    for (auto& e : ev) GF_CUDA(cudaEventCreate(&e));
    GF_CUDA(cudaEventRecord(ev[0], st));
  }
  {
    const unsigned gx = (unsigned)ceil_div(q, 256);
    const unsigned gy = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div((int64_t)num_sms() * 8, gx), m));
    colmax_f64_kernel<<<dim3(gx, gy), 256, 0, st>>>((const double*)A->data, m, A->ld, q, cmax);
    GF_CHECK_LAUNCH();
    colexp_kernel<<<(unsigned)ceil_div(q, 256), 256, 0, st>>>(cmax, q, ex);
    GF_CHECK_LAUNCH();
    slice_i8_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nkb * ncp, 256), num_sms() * 16), 256, 0, st>>>(
        (const double*)A->data, m, A->ld, q, ncp, nkb, cmax, (uint4*)scratch, (int64_t)(slice_bytes / 16));
    GF_CHECK_LAUNCH();
  }
  if (verbose) GF_CUDA(cudaEventRecord(ev[1], st));
  static bool attr = false;
  if (!attr) {
    GF_CUDA(cudaFuncSetAttribute(syrk_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, I8_SMEM));
    attr = true;
  }
  syrk_i8_kernel<<<(unsigned)tl.size(), I8_THREADS, I8_SMEM, st>>>(tmA, tmB, nkb, q, d_tiles, ex, G, ldg);
  GF_CHECK_LAUNCH();
  upper_to_lower<<<dim3((unsigned)ceil_div(q, 32), (unsigned)ceil_div(q, 8)), dim3(32, 8), 0, st>>>(G, q, ldg);
  GF_CHECK_LAUNCH();
  if (verbose) {
    GF_CUDA(cudaEventRecord(ev[2], st));
    GF_CUDA(cudaStreamSynchronize(st));
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    fprintf(stderr, "[gf] gram fp64 int8 slices: slice %.2f ms, syrk %.2f ms (%zu tiles)\n", a, b, tl.size());
    for (auto& e : ev) cudaEventDestroy(e);
  }
  GF_CUDA(cudaStreamSynchronize(st));   // `small` is freed on return
  return true;
}

}  // namespace gf
