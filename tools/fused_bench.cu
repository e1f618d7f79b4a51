// Dev microbenchmark for the fused row/column kernel (gf_fused.cuh) on the
// bench shape: times it with a trivial epilogue, with a YEpi-like fp64
// epilogue (square prox, numpy-rounded divisions), and a stream-only ring
// (TMA into the smem ring, consumers release rows without math) that bounds
// what this pipeline shape can pull from HBM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -I paper_1503_08366_b200/csrc tools/fused_bench.cu -o tools/fused_bench
//   tools/fused_bench [m n reps]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <functional>

#include "gf_fused.cuh"
#include "gf_terms.cuh"

using namespace gf;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

struct Flag {
  int status;
};

struct DummyEpi {
  static constexpr int NR = 4;
  const Flag* fl;
  double* out;
  struct RowIn {
    double a;
  };
  __device__ bool active() const { return fl->status == 0; }
  __device__ void begin() {}
  __device__ RowIn load_in(int64_t i) const { return RowIn{0.0}; }
  struct Mid {
    double a;
  };
  __device__ Mid mid(const RowIn& in, const double* dots, double& w0, double& w1) const {
    w0 = dots[0] * 0.5;
    w1 = dots[1];
    return Mid{dots[0]};
  }
  __device__ void tail(int64_t i, const RowIn& in, const double* dots, const Mid& r, double* red,
                       unsigned& flags) const {
    red[0] += r.a;
  }
};

// YEpi-like: same loads, divisions, prox and stores as gf_solver.cu YEpi (k>0 path).
// LOADS=false: the per-row inputs are synthesised (no global loads), STORES=false: no stores.
template <bool LOADS, bool STORES>
struct HeavyEpiT {
  static constexpr int NR = 4;
  const Flag* fl;
  TermsView f;
  const double* d;
  double *yk, *yt, *cy, *yh2, *nuh2;
  double rho, ratio, alpha;
  struct RowIn {
    double di, cy, yk, yt;
    Term t;
  };
  __device__ bool active() const { return fl->status == 0; }
  __device__ void begin() {}
  __device__ RowIn load_in(int64_t i) const {
    RowIn in;
    if (!LOADS) {
      in.di = 1.0 + 1e-9 * (double)i;
      in.cy = 0.0;
      in.yk = 0.0;
      in.yt = 0.0;
      in.t = Term{1, 1.0, 0.0, 1.0, 0.0, 0.0};
      return in;
    }
    in.di = d[i];
    in.cy = cy[i];
    in.yk = yk[i];
    in.yt = yt[i];
    in.t = load_term(f, i);
    return in;
  }
  struct Mid {
    double ykv, ytv, yh, yhh, nu, cyn;
  };
  __device__ Mid mid(const RowIn& in, const double* dots, double& w0, double& w1) const {
    Mid r;
    r.ykv = dots[0];
    r.ytv = M_(S_(in.cy, r.ykv), ratio);
    const double di = in.di;
    r.yh = prox_term(in.t, M_(rho, M_(di, di)), D_(S_(r.ykv, r.ytv), di));
    r.yhh = M_(r.yh, di);
    r.nu = M_(-rho, A_(S_(r.yhh, r.ykv), r.ytv));
    const double ry = A_(M_(alpha, r.yhh), M_(S_(1.0, alpha), r.ykv));
    r.cyn = A_(ry, r.ytv);
    w0 = r.cyn * 1e-3;
    w1 = r.nu * 1e-3;
    return r;
  }
  __device__ void tail(int64_t i, const RowIn& in, const double* dots, const Mid& r, double* red,
                       unsigned& flags) const {
    if (!isfinite(r.yh)) flags |= 1;
    if (STORES) {
    yk[i] = r.ykv;
    yt[i] = r.ytv;
    yh2[i] = r.yh;
    nuh2[i] = r.nu;
    cy[i] = r.cyn;
    }
    const double rp = S_(D_(dots[1], in.di), r.yh);
    red[0] += rp * rp;
    red[1] += r.yh * r.yh;
    red[2] += eval_term(in.t, r.yh);
    red[3] += (r.yhh - r.ykv) * (r.yhh - r.ykv);
  }
};
using HeavyEpi = HeavyEpiT<true, true>;
using HeavyNoLoad = HeavyEpiT<false, true>;
using HeavyNoStore = HeavyEpiT<true, false>;

// Stream-only ring: producer TMA fills slots, 16 consumer warps wait and release.
constexpr int kFusedWarps = 16;
constexpr int kProdWarp = 18;
constexpr int kFusedAll = fused_threads(16);
__global__ void __launch_bounds__(kFusedAll, 1)
stream_ring(const float* A, int64_t rows, int64_t ld, int nslot, float* sink) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxSlots], sfree[kMaxSlots];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned rb = (unsigned)(ld * 4);
  const int64_t r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  const int nr = (int)(r1 - r0);
  if (tid == 0) {
    for (int s = 0; s < nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sfree[s], kFusedWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kProdWarp) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int slot = 0;
      for (int j = 0; j < nr; ++j) {
        if (j >= nslot) mbar_wait(&sfree[slot], (unsigned)(((j / nslot) - 1) & 1));
        mbar_arrive_expect_tx(&full[slot], rb);
        bulk_g2s(smem_raw + slot * rb, A + (r0 + j) * ld, rb, &full[slot], pol);
        if (++slot == nslot) slot = 0;
      }
    }
    return;
  }
  if (warp >= kFusedWarps) return;
  int slot = 0;
  unsigned ph = 0;
  float acc = 0.f;
  for (int j = 0; j < nr; ++j) {
    mbar_wait(&full[slot], ph);
    acc += reinterpret_cast<const float*>(smem_raw + slot * rb)[tid];
    __syncwarp();
    if (lane == 0) mbar_arrive_expect_tx(&sfree[slot], 0);
    if (++slot == nslot) { slot = 0; ph ^= 1u; }
  }
  if (acc == 12345.f) sink[tid] = acc;
}

// Epilogue chain alone: `busy` extra warps spin on FFMA+LDS while warp 0 runs
// the YEpi-like epilogue over `groups` groups of 2 rows; returns cycles/group.
template <class Epi>
__global__ void epi_alone(Epi epi, int groups, int busy_iters, unsigned long long* out, float* sink) {
  __shared__ float buf[4096];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp > 0) {
    float a = lane, b = 1.0001f;
    for (int i = 0; i < busy_iters; ++i) {
      float4 v = reinterpret_cast<float4*>(buf)[(threadIdx.x + i) & 1023];
      a = fmaf(a, b, v.x); a = fmaf(a, b, v.y); a = fmaf(a, b, v.z); a = fmaf(a, b, v.w);
      a = fmaf(a, b, v.x); a = fmaf(a, b, v.y); a = fmaf(a, b, v.z); a = fmaf(a, b, v.w);
    }
    if (a == 1234.f) sink[threadIdx.x] = a;
    return;
  }
  double ered[4] = {0, 0, 0, 0};
  unsigned fl = 0;
  typename Epi::RowIn in = epi.load_in(lane);
  long long t0 = clock64();
  for (int g = 0; g < groups; ++g) {
    double v[4];
    for (int q = 0; q < 4; ++q) v[q] = lane < 16 ? 0.01 * (lane + q + g) : 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o, 16);
    double dots[2] = {lane == 0 ? v[0] : v[2], lane == 0 ? v[1] : v[3]};
    if (lane < 2) {
      double w0, w1;
      auto md = epi.mid(in, dots, w0, w1);
      buf[lane] = (float)w0;
      buf[lane + 2] = (float)w1;
      epi.tail(2 * g + lane, in, dots, md, ered, fl);
    }
    __syncwarp();
    in = epi.load_in(2 * g + 4 + lane);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (ered[0] == 1234.0) sink[0] = (float)ered[1];
}

template <typename Epi, int NV, int TR, int CW>
float time_fused(const float* A, int64_t m, int64_t ld, const float* x0, const float* x1, Epi epi, int nslot,
                 double* rpart, double* cpart, int reps, size_t smem) {
  auto k = fused_rowcol_kernel<float, NV, TR, CW, Epi>;
  {  // this instance's lane-partial buffers sit in front of the ring
    const size_t red = (size_t)fused_epi(CW) * CW * 32 * 2 * TR * 4, rb = (size_t)ld * 4;
    while (nslot > 3 * TR + 1 && red + nslot * rb > 227 * 1024 - 2048) --nslot;
    smem = red + nslot * rb;
  }
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) k<<<148, fused_threads(CW), smem>>>(A, m, ld, x0, x1, epi, nslot, rpart, cpart);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) k<<<148, fused_threads(CW), smem>>>(A, m, ld, x0, x1, epi, nslot, rpart, cpart);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
#ifdef GF_FUSED_TRACE
  // one traced launch: per-CTA cycle counters
  std::vector<unsigned long long> zero(148 * 16, 0), tr(148 * 16);
  CK(cudaMemcpyToSymbol(gf_fused_trace, zero.data(), zero.size() * 8));
  k<<<148, fused_threads(CW), smem>>>(A, m, ld, x0, x1, epi, nslot, rpart, cpart);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpyFromSymbol(tr.data(), gf_fused_trace, tr.size() * 8));
  double acc[16] = {0};
  for (int c = 0; c < 148; ++c)
    for (int j = 0; j < 16; ++j) acc[j] += (double)tr[c * 16 + j] / 148.0 / 1965.0;   // us per CTA
  const double groups = (double)m / 148 / TR;
  printf("   per CTA (us): epi wait redf %.1f+%.1f | reduce %.1f | wait we %.1f | mid %.1f | tail+load %.1f | "
         "epi total %.1f ;  compute w0: wait full %.1f rede %.1f wf %.1f ; producer wait sfree %.1f  (groups %.0f, per group epi %.2f us)\n",
         acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], acc[6], acc[8], acc[9], acc[10], acc[11], groups,
         (acc[2] + acc[3] + acc[4] + acc[5]) / groups);
#endif
  return ms / reps;
}

int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 200000;
  const int64_t n = argc > 2 ? atoll(argv[2]) : 5000;
  const int reps = argc > 3 ? atoi(argv[3]) : 20;
  const int64_t ld = (n + 31) / 32 * 32;
  float* A;
  CK(cudaMalloc(&A, m * ld * 4));
  {
    std::vector<float> h(ld * 1024);
    for (auto& v : h) v = (float)(rand() % 1000) / 1000.f - 0.5f;
    for (int64_t r = 0; r < m; r += 1024)
      CK(cudaMemcpy(A + r * ld, h.data(), std::min<int64_t>(1024, m - r) * ld * 4, cudaMemcpyHostToDevice));
  }
  float *x0, *x1, *sink;
  CK(cudaMalloc(&x0, ld * 4));
  CK(cudaMalloc(&x1, ld * 4));
  CK(cudaMalloc(&sink, 4096 * 4));
  CK(cudaMemset(x0, 0, ld * 4));
  CK(cudaMemset(x1, 0, ld * 4));
  double *rpart, *cpart, *vec;
  CK(cudaMalloc(&rpart, 148 * 8 * 8 * 8));
  CK(cudaMalloc(&cpart, 148 * 2 * ld * 8));
  CK(cudaMalloc(&vec, 8 * m * 8));
  CK(cudaMemset(vec, 0, 8 * m * 8));
  Flag* fl;
  CK(cudaMalloc(&fl, sizeof(Flag)));
  CK(cudaMemset(fl, 0, sizeof(Flag)));
  int8_t* h;
  CK(cudaMalloc(&h, m));
  CK(cudaMemset(h, 1, m));   // kSquare
  double* ones;
  CK(cudaMalloc(&ones, m * 8));
  {
    std::vector<double> o(m, 1.0);
    CK(cudaMemcpy(ones, o.data(), m * 8, cudaMemcpyHostToDevice));
  }
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
  FusedPlan p = plan_fused(m, ld, 4, 148, (size_t)optin);
  printf("plan: nv %d nslot %d tr %d smem %zu\n", p.nv, p.nslot, p.tr, p.smem);
  const double gb = (double)m * n * 4 / 1e9;

  CK(cudaFuncSetAttribute(stream_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  for (int ns : {3, 4, 5, 6, 8}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) stream_ring<<<148, kFusedAll, p.smem>>>(A, m, ld, ns, sink);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) stream_ring<<<148, kFusedAll, p.smem>>>(A, m, ld, ns, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    printf("stream_ring nslot %2d  %.4f ms  %.0f GB/s\n", ns, ms, gb / ms * 1e3);
  }
  DummyEpi de{fl, vec};
  HeavyEpi he{fl, TermsView{h, ones, vec, ones, vec, vec}, ones, vec, vec + m, vec + 2 * m, vec + 3 * m,
              vec + 4 * m, 1.0, 1.0, 1.7};
  HeavyNoLoad hn{fl, TermsView{h, ones, vec, ones, vec, vec}, ones, vec, vec + m, vec + 2 * m, vec + 3 * m,
                 vec + 4 * m, 1.0, 1.0, 1.7};
  HeavyNoStore hs{fl, TermsView{h, ones, vec, ones, vec, vec}, ones, vec, vec + m, vec + 2 * m, vec + 3 * m,
                  vec + 4 * m, 1.0, 1.0, 1.7};
  {
    unsigned long long* out;
    CK(cudaMalloc(&out, 148 * 8));
    for (int busy : {0, 4, 16}) {
      for (int it = 0; it < 2; ++it) epi_alone<HeavyEpi><<<148, 32 * (1 + busy)>>>(he, 600, busy ? 200000 : 0, out, sink);
      CK(cudaDeviceSynchronize());
      unsigned long long c;
      CK(cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost));
      printf("epilogue alone, %2d busy warps: %.0f cycles per group\n", busy, (double)c / 600);
    }
    for (int busy : {0, 16}) {
      epi_alone<HeavyNoLoad><<<148, 32 * (1 + busy)>>>(hn, 600, busy ? 200000 : 0, out, sink);
      CK(cudaDeviceSynchronize());
      unsigned long long c;
      CK(cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost));
      printf("epilogue alone (no loads), %2d busy warps: %.0f cycles per group\n", busy, (double)c / 600);
    }
  }
  // configurations timed round-robin (clock / power drift hits all alike);
  // min and median over rounds
  struct Cfg { const char* name; std::function<float()> run; std::vector<float> t; };
  std::vector<Cfg> cfgs;
#define ADD(EPI, e, NV, TR, CW)                                                                          \
  cfgs.push_back({#EPI " NV=" #NV " CW=" #CW, [&]() {                                                    \
    return time_fused<EPI, NV, TR, CW>(A, m, ld, x0, x1, e, p.nslot, rpart, cpart, reps, p.smem); }, {}});
  ADD(DummyEpi, de, 5, 2, 8)
  ADD(DummyEpi, de, 4, 2, 12)
  ADD(HeavyEpi, he, 5, 2, 8)
  ADD(HeavyEpi, he, 4, 2, 12)
  const int rounds = argc > 4 ? atoi(argv[4]) : 5;
  for (int r = 0; r < rounds; ++r)
    for (auto& c : cfgs) c.t.push_back(c.run());
  for (auto& c : cfgs) {
    std::sort(c.t.begin(), c.t.end());
    printf("fused %-22s NE=%d  min %.4f ms (%.0f GB/s)  median %.4f ms\n", c.name, fused_epi(8), c.t[0],
           gb / c.t[0] * 1e3, c.t[c.t.size() / 2]);
  }
  return 0;
}
