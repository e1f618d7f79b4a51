// Sanitizer calibration: the mbarrier hand-off patterns of gf_fused.cuh in a
// trivially correct kernel, one variant per launch, so that compute-sanitizer
// synccheck / racecheck reports on the real kernels can be told apart from
// tool limitations.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -I paper_1503_08366_b200/csrc tools/san/mbar_sanity.cu -o tools/san/mbar_sanity
//   compute-sanitizer --tool synccheck tools/san/mbar_sanity V
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include "gf_fused.cuh"
using namespace gf;

__device__ __forceinline__ void arrive_generic(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool try_wait_nohint(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool test_wait(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

// warp 0 (producer of data) -> warp 1 (consumer), ROUNDS rounds, one barrier
// pair (full: 1 arrival from warp 0; empty: 1 arrival from warp 1)
template <int V>
__global__ void handoff(int* out, int rounds) {
  __shared__ __align__(8) uint64_t full, empty;
  __shared__ int buf[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&full, 1);
    mbar_init(&empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int acc = 0;
  for (int r = 0; r < rounds; ++r) {
    const unsigned ph = r & 1;
    if (warp == 0) {
      if (r > 0) {
        if (V == 0 || V == 2) mbar_wait(&empty, ph ^ 1u);
        else if (V == 1) mbar_wait_u32(smem_u32(&empty), ph ^ 1u);
        else if (V == 3) { while (!try_wait_nohint(&empty, ph ^ 1u)) {} }
        else { while (!test_wait(&empty, ph ^ 1u)) {} }
      }
      buf[lane] = r * 32 + lane;
      __syncwarp();
      if (lane == 0) {
        if (V == 0) mbar_arrive_u32(smem_u32(&full));
        else if (V == 2) mbar_arrive_expect_tx(&full, 0);
        else arrive_generic(&full);
      }
    } else if (warp == 1) {
      if (V == 0 || V == 2) mbar_wait(&full, ph);
      else if (V == 1) mbar_wait_u32(smem_u32(&full), ph);
      else if (V == 3) { while (!try_wait_nohint(&full, ph)) {} }
      else { while (!test_wait(&full, ph)) {} }
      acc += buf[lane];
      __syncwarp();
      if (lane == 0) {
        if (V == 0) mbar_arrive_u32(smem_u32(&empty));
        else if (V == 2) mbar_arrive_expect_tx(&empty, 0);
        else arrive_generic(&empty);
      }
    }
  }
  if (warp == 1) out[lane] = acc;
}


// Variants 5-7: the fused kernel's shape -- arrays of barriers initialised in a
// loop by thread 0, NE consumer warps each waiting on barrier [warp - NP]
// (runtime index), NP producer warps arriving on a u32 address; 6 adds a large
// dynamic shared-memory ring, 7 also a griddepcontrol.wait before the waits.
// Variants 8 / 9: 26 / 27 extra barriers initialised first, so that the six
// used ones are the 27th-32nd / 28th-33rd of the CTA (does the tool track a
// bounded number of mbarriers per CTA?).
template <int V>
__global__ void handoff_arr(int* out, int rounds, int ne) {
  constexpr int NP = 4;
  constexpr int NFULL = V == 8 ? 26 : (V == 9 ? 27 : 32);
  extern __shared__ __align__(128) unsigned char dyn[];
  __shared__ __align__(8) uint64_t full[32], redf[3], rede[3];
  __shared__ int buf[3][NP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NFULL; ++s) mbar_init(&full[s], 1);
    for (int b = 0; b < ne; ++b) {
      mbar_init(&redf[b], NP);
      mbar_init(&rede[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (V >= 6 && threadIdx.x == 0) dyn[1000] = 1;
  if (V == 7) pdl_wait();
  int acc = 0;
  if (warp < NP) {
    const uint32_t redf0 = smem_u32(redf), rede0 = smem_u32(rede);
    for (int r = 0; r < rounds; ++r) {
      const int b = r % ne;
      const unsigned use = r / ne;
      if (use >= 1) mbar_wait_u32(rede0 + 8u * b, (use - 1) & 1u);
      if (lane == 0) buf[b][warp] = r + warp;
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(redf0 + 8u * b);
    }
  } else if (warp < NP + ne) {
    const int b = warp - NP;
    for (int r = b; r < rounds; r += ne) {
      const unsigned use = r / ne;
      mbar_wait_u32(smem_u32(&redf[b]), use & 1u);
      int v = lane < NP ? buf[b][lane] : 0;
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&rede[b], 0);
      acc += v;
    }
  }
  if (warp == NP) out[lane] = acc;
}

int main(int argc, char** argv) {
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  int* out;
  cudaMalloc(&out, 32 * sizeof(int));
  switch (v) {
    case 0: handoff<0><<<2, 64>>>(out, 64); break;
    case 1: handoff<1><<<2, 64>>>(out, 64); break;
    case 2: handoff<2><<<2, 64>>>(out, 64); break;
    case 3: handoff<3><<<2, 64>>>(out, 64); break;
    case 4: handoff<4><<<2, 64>>>(out, 64); break;
    case 5: handoff_arr<5><<<2, 7 * 32>>>(out, 64, 3); break;
    case 6:
      cudaFuncSetAttribute(handoff_arr<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      handoff_arr<6><<<2, 7 * 32, 200 * 1024>>>(out, 64, 3);
      break;
    case 8: handoff_arr<8><<<2, 7 * 32>>>(out, 64, 3); break;
    case 9: handoff_arr<9><<<2, 7 * 32>>>(out, 64, 3); break;
    default:
      cudaFuncSetAttribute(handoff_arr<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      handoff_arr<7><<<2, 7 * 32, 200 * 1024>>>(out, 64, 3);
      break;
  }
  cudaError_t e = cudaDeviceSynchronize();
  int h[32];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  // sum over r of (32 r + lane) for lane 0: 32 * 64*63/2
  if (v < 5) printf("variant %d: %s, out[0] = %d (expect %d)\n", v, cudaGetErrorString(e), h[0], 32 * 64 * 63 / 2);
  else printf("variant %d: %s, out[0] = %d (expect %d)\n", v, cudaGetErrorString(e), h[0], 4 * (22 * 21 / 2 * 3 + 0) + 0);
  return 0;
}
