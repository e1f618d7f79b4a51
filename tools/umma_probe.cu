// Dev probe: one tcgen05.mma kind::tf32 (M=128, N=16, K=8) with A/B in shared
// memory in a chosen layout; prints max error vs a CPU reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -o umma_probe tools/umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

constexpr int M = 128, N = 16, K = 8;

// mode 0: MN-major no-swizzle (core = 8 k-rows x 4 mn elems), SBO = mn-group stride 128 B
// mode 1: K-major no-swizzle (core = 8 mn-rows x 4 k elems), SBO = mn-group(8 rows) stride,
//         LBO = k-chunk stride
__global__ void probe(const float* A, const float* B, float* D, int mode, int swap) {
  __shared__ __align__(1024) float sa[M * K];
  __shared__ __align__(1024) float sb[N * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid >> 5;
  // fill: A is M x K (A[m][k]), B is N x K (B[n][k])
  for (int idx = tid; idx < M * K; idx += blockDim.x) {
    int m = idx / K, k = idx % K;
    int off;
    if (mode == 0) off = (m / 4) * 32 + k * 4 + (m % 4);                 // floats: group*128B + krow*16B + e
    else off = (k / 4) * (M * 4) + (m / 8) * 32 + (m % 8) * 4 + (k % 4);  // kchunk*LBO + mngroup*128B + row*16B + e
    sa[off] = A[idx];
  }
  for (int idx = tid; idx < N * K; idx += blockDim.x) {
    int n = idx / K, k = idx % K;
    int off;
    if (mode == 0) off = (n / 4) * 32 + k * 4 + (n % 4);
    else off = (k / 4) * (N * 4) + (n / 8) * 32 + (n % 8) * 4 + (k % 4);
    sb[off] = B[idx];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = tbase;
  if (tid == 0) {
    uint64_t da, db;
    if (mode == 0) {
      uint32_t lboA = (M / 4) * 128, lboB = (N / 4) * 128;
      da = swap ? sdesc(su32(sa), 128, lboA) : sdesc(su32(sa), lboA, 128);
      db = swap ? sdesc(su32(sb), 128, lboB) : sdesc(su32(sb), lboB, 128);
    } else {
      da = swap ? sdesc(su32(sa), 128, M * 16) : sdesc(su32(sa), M * 16, 128);
      db = swap ? sdesc(su32(sb), 128, N * 16) : sdesc(su32(sb), N * 16, 128);
    }
    uint32_t major = mode == 0 ? 1u : 0u;
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (major << 15) | (major << 16) |
                     ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
        "l"(da), "l"(db), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[16];
  uint32_t taddr = tm + ((uint32_t)(warp * 32) << 16);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                 "=r"(v[15])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int j = 0; j < 16; ++j) D[tid * N + j] = __uint_as_float(v[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N), R(M * N);
  for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 7) % 11 - 5);
  for (int i = 0; i < N * K; ++i) B[i] = (float)((i * 5) % 7 - 3);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += A[m * K + k] * B[n * K + k];
      R[m * N + n] = (float)s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode)
    for (int swap = 0; swap < 2; ++swap) {
      cudaMemset(dD, 0, D.size() * 4);
      probe<<<1, 128>>>(dA, dB, dD, mode, swap);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0, mx = 0;
      for (int i = 0; i < M * N; ++i) { err = fmax(err, fabs(D[i] - R[i])); mx = fmax(mx, fabs(D[i])); }
      printf("mode %d (%s) swap %d: err %s max|err| %.3g max|D| %.3g  D[0][0..3] %g %g %g %g ref %g %g %g %g\n", mode,
             mode == 0 ? "MN-major" : "K-major", swap, cudaGetErrorString(e), err, mx, D[0], D[1], D[2], D[3], R[0],
             R[1], R[2], R[3]);
    }
  return 0;
}
