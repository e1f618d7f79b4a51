// Tensor-core Gram matrix G = A'A for fp32 A (tall projector setup),
// tcgen05 kind::tf32 with a 3xTF32 split for fp32-grade accuracy.
//
// Reference: projection.py:86-90 (gram = A.T @ A; gram += I) on OpenBLAS dgemm.
// The north star asks for a tensor-core SYRK; plain TF32 perturbs G enough to
// move fp32 iterates (x error 3.5e-4 on SVM) and BF16 changes
// iteration counts, so each fp32 element is split as a = hi + lo with
// hi = tf32(a), lo = tf32(a - hi) and
//     G += hi_i' hi_j + hi_i' lo_j + lo_i' hi_j           (3 MMAs)
// which keeps ~22 mantissa bits.  The accumulator lives in TMEM in fp32 and is
// drained into the fp64 G every `kchunk` rows: the tensor core's fp32
// accumulation truncates, so its relative error grows with the number of
// accumulate steps per drain (measured ~3e-8 per step); the drain interval
// bounds it while the long reduction over m = 2e5 rows is carried in fp64.
//
// Tile: 128 columns of A (MMA M) x 256 columns (MMA N), lower-triangle tiles
// only (G is mirrored afterwards).  Warp roles (416 threads):
//   warps 0-3   epilogue: tcgen05.ld the 128x256 fp32 accumulator, add into G (fp64)
//   warp 4      TMEM allocator + MMA issuer (one thread)
//   warps 5-12  producers: coalesced column loads of 4 fp32 rows, split into
//               hi/lo, one 16-byte store each into the K-major no-swizzle
//               core-matrix layout the MMA descriptors expect
// Pipelines: 4 shared-memory stages (full/empty mbarriers; empty is signalled
// by tcgen05.commit) and 2 TMEM accumulators (256 columns each; full by
// tcgen05.commit, empty by the epilogue warps).

#include <cuda.h>
#include <cudaTypedefs.h>

#include "gf_internal.h"

namespace gf {
namespace syrk {

// K-major, no-swizzle operand layout (verified on B200 with tools/umma_probe.cu):
// a core matrix is 8 MN-rows x 16 bytes (4 tf32 along K), 128 contiguous
// bytes; 8-row groups are SBO = 128 B apart, 4-element K chunks LBO apart.
constexpr int TM = 128, TN = 256, BK = 16, NST = 2;
// rows per TMEM accumulation: 1024 -> max |G error| / max |G| ~ 9.5e-6 on a
// 20000 x 1300 Gaussian matrix (512: 4.7e-6, 128: 1.2e-6; tools/syrk_accuracy.py);
// 1024 halves the fp64 drain traffic of 512 (Gram 39 -> 29 ms at 200000 x 5000)
constexpr int KCHUNK_DEFAULT = 1024;
constexpr int A_BYTES = (BK / 4) * (TM / 8) * 128; // 8 KB per hi/lo
constexpr int B_BYTES = (BK / 4) * (TN / 8) * 128; // 16 KB per hi/lo
constexpr int LBO_A = (TM / 8) * 128;              // K-chunk stride
constexpr int LBO_B = (TN / 8) * 128;
constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;   // 48 KB
constexpr int NPROD = 8;                           // converter warps
constexpr int LOADER_WARP = 5 + NPROD;             // TMA loader warp
constexpr int THREADS = (6 + NPROD) * 32;
// raw fp32 ring filled by 2-D tensor TMA: per stage two boxes, BK rows x TM
// columns (A panel, 8 KB) then BK rows x TN columns (B panel, 16 KB), rows
// and columns past the matrix zero-filled by the TMA unit
constexpr int RAW_A = BK * TM * 4;
constexpr int RAW_BYTES = BK * (TM + TN) * 4;      // 24 KB
constexpr int NRAW = 5;
constexpr int SMEM = NST * STAGE + NRAW * RAW_BYTES;   // 96 + 120 KB

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

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = 256.
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                           ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
               : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
syrk_tf32x3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t K,
                   int64_t q, int64_t kchunk, const int2* __restrict__ tiles, double* __restrict__ G, int64_t ldg) {
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
    constexpr int NITEM = ((BK / 4) * (TM + TN)) / (NPROD * 32);   // 6
    const int pt = tid - 5 * 32;   // 0..255
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
        float f[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) f[e] = col[(4 * kc + e) * w];
        uint4 hi, lo;
        hi.x = to_tf32(f[0]); lo.x = to_tf32(f[0] - __uint_as_float(hi.x));
        hi.y = to_tf32(f[1]); lo.y = to_tf32(f[1] - __uint_as_float(hi.y));
        hi.z = to_tf32(f[2]); lo.z = to_tf32(f[2] - __uint_as_float(hi.z));
        hi.w = to_tf32(f[3]); lo.w = to_tf32(f[3] - __uint_as_float(hi.w));
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
          for (int kk = 0; kk < BK / 8; ++kk) {
            // one MMA covers K = 8 = two 4-element K chunks
            const uint64_t dah = smem_desc(a_hi + 2 * kk * LBO_A, LBO_A, 128);
            const uint64_t dal = smem_desc(a_lo + 2 * kk * LBO_A, LBO_A, 128);
            const uint64_t dbh = smem_desc(b_hi + 2 * kk * LBO_B, LBO_B, 128);
            const uint64_t dbl = smem_desc(b_lo + 2 * kk * LBO_B, LBO_B, 128);
            const uint32_t accum = (it > it0 || kk > 0) ? 1u : 0u;
            mma_tf32(d, dah, dbh, accum);
            mma_tf32(d, dah, dbl, 1u);
            mma_tf32(d, dal, dbh, 1u);
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
    for (int64_t c = 0; c < nchunks; ++c) {
      const int acc = (int)(c & 1);
      bar_wait(&accf[acc], (unsigned)((c >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int cc = 0; cc < TN / 32; ++cc) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * TN + cc * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // G is symmetric: accumulate the tile's transpose, G[j][i], so the 32
        // lanes (consecutive i) touch 256 contiguous bytes per instruction;
        // the upper triangle is mirrored down afterwards (gram_finish).
        // all 32 loads are issued before any store (a plain `+=` loop would
        // serialize on possible aliasing between the stores and later loads)
        // (two halves of 16: 32 fp64 values plus the 32 accumulator words
        // overflowed the 128-register budget into local memory)
        if (i < q) {
          const int64_t jn = min((int64_t)32, q - (j0 + cc * 32));
          double* col = G + (j0 + cc * 32) * ldg + i;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double g[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) g[t] = 16 * h + t < jn ? col[(16 * h + t) * ldg] : 0.0;
#pragma unroll
            for (int t = 0; t < 16; ++t)
              if (16 * h + t < jn) col[(16 * h + t) * ldg] = g[t] + (double)__uint_as_float(v[16 * h + t]);
          }
        }
      }
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

// G (fp64, zeroed by the caller) += A'A for fp32 A (m x ld, columns >= n zero).
void gram_tf32x3(const gf_matrix* A, double* G, int64_t ldg, cudaStream_t st) {
  using namespace syrk;
  const int64_t q = A->n;
  const int64_t bi_n = ceil_div(q, TM), bj_n = ceil_div(q, TN);
  std::vector<int2> tl;
  for (int64_t bi = 0; bi < bi_n; ++bi)
    for (int64_t bj = 0; bj < bj_n; ++bj)
      if (2 * bj <= bi) tl.push_back(make_int2((int)bi, (int)bj));   // lower-triangle tiles
  DBuf d_tiles(tl.size() * sizeof(int2));
  GF_CUDA(cudaMemcpyAsync(d_tiles.p, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  static bool attr = false;
  if (!attr) {
    GF_CUDA(cudaFuncSetAttribute(syrk_tf32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    attr = true;
  }
  const char* kc_env = getenv("GF_SYRK_KCHUNK");
  int64_t kchunk = kc_env ? std::max<int64_t>(BK, atoll(kc_env) / BK * BK) : KCHUNK_DEFAULT;
  const CUtensorMap tmA = panel_map(A, TM), tmB = panel_map(A, TN);
  syrk_tf32x3_kernel<<<(unsigned)tl.size(), THREADS, SMEM, st>>>(tmA, tmB, A->m, q, kchunk, d_tiles.as<int2>(), G,
                                                                 ldg);
  GF_CHECK_LAUNCH();
  upper_to_lower<<<dim3((unsigned)ceil_div(q, 32), (unsigned)ceil_div(q, 8)), dim3(32, 8), 0, st>>>(G, q, ldg);
  GF_CHECK_LAUNCH();
  GF_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gf
