// Shared device/host helpers for the graphform-b200 CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include <string>

#include "../../include/graphform_b200.h"

namespace gf {

// ----------------------------------------------------------------- errors --
// Thread-local last-error message; every C-ABI entry point returns a GF_*
// code and leaves the message here (gf_last_error()).
void set_error(const std::string& msg);
const char* last_error();

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void throw_error(int code, const std::string& msg);

#define GF_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      ::gf::throw_error(GF_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define GF_CHECK_LAUNCH() GF_CUDA(cudaGetLastError())

#define GF_REQUIRE(cond, code, msg)         \
  do {                                      \
    if (!(cond)) ::gf::throw_error(code, msg); \
  } while (0)

// ------------------------------------------------------------------ device --
int num_sms();  // SM count of the current device (148 on B200)

constexpr int kWarp = 32;

template <typename T>
struct Vec16;  // 16-byte vector of T
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int n = 4;
};
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int n = 2;
};

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in
// the stream drains; pdl_wait() blocks until the predecessor has completed
// and its writes are visible (a no-op without the attribute), and
// pdl_trigger() lets the successor start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ float vget(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}
__device__ __forceinline__ double vget(const double2& v, int i) { return i == 0 ? v.x : v.y; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned warp_or(unsigned v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Streaming 16-byte load that does not allocate in L1 (A is read once).
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

// Row stride (elements) of every matrix the library stores: 128-byte aligned
// rows, so each row start is valid for 16-byte vector loads and TMA bulk
// copies, and the zero padding contributes nothing to any product.
inline int64_t padded_ld(int64_t n, int dtype) {
  return round_up(n > 0 ? n : 1, dtype == GF_F32 ? 32 : 16);
}

}  // namespace gf
