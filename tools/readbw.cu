// Dev probe: what a read-only stream over a 4 GB buffer reaches on this GPU
// (the ceiling for the fused iteration kernel, which only reads A_hat), next to
// the D2D copy bandwidth that MEASURED_PEAKS.json records.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/readbw.cu -o tools/readbw
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

template <int U>
__global__ void read_kernel(const float4* __restrict__ a, long long n4, float* sink) {
  float acc = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < n4; i += stride) {
    float4 v = __ldcs(a + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5f) sink[0] = acc;
}

// contiguous chunk per CTA (the fused kernel's row-range shape)
template <int U>
__global__ void read_chunk_kernel(const float4* __restrict__ a, long long n4, float* sink) {
  const long long c0 = n4 * blockIdx.x / gridDim.x, c1 = n4 * (blockIdx.x + 1) / gridDim.x;
  float acc = 0.f;
  long long i = c0 + threadIdx.x;
  for (; i + (U - 1) * blockDim.x < c1; i += U * blockDim.x) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < c1; i += blockDim.x) {
    float4 v = __ldcs(a + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5f) sink[0] = acc;
}

template <class F>
float timeit(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const long long bytes = 4000000000LL;
  const long long n4 = bytes / 16;
  float4 *a, *b;
  float* sink;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(a, 0, bytes));
  const double gb = bytes / 1e9;
  float ms = timeit([&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); }, 10);
  printf("D2D copy      %.3f ms  %.0f GB/s (read+write)\n", ms, 2 * gb / ms * 1e3);
  for (int bpsm : {1, 2, 4, 8}) {
    for (int th : {256, 512, 1024}) {
      if (bpsm * th > 2048) continue;
      ms = timeit([&] { read_kernel<4><<<148 * bpsm, th>>>(a, n4, sink); }, 10);
      printf("read gridstride U4 %4d x %4d  %.3f ms  %.0f GB/s\n", 148 * bpsm, th, ms, gb / ms * 1e3);
      ms = timeit([&] { read_chunk_kernel<4><<<148 * bpsm, th>>>(a, n4, sink); }, 10);
      printf("read chunk      U4 %4d x %4d  %.3f ms  %.0f GB/s\n", 148 * bpsm, th, ms, gb / ms * 1e3);
    }
  }
  ms = timeit([&] { read_kernel<8><<<148 * 2, 1024>>>(a, n4, sink); }, 10);
  printf("read gridstride U8  296 x 1024  %.3f ms  %.0f GB/s\n", ms, gb / ms * 1e3);
  return 0;
}
