// Input synthesis on the device: numpy's Generator(PCG64).normal, bit for bit.
//
// The reference builds every instance with numpy streams
// (generators.py:80-264: A = rng.normal(...) for each family).  At the paper's
// 1e9-coefficient scale that host generation takes ~25 s plus a 4-8 GB H2D
// copy.  This file reproduces the same draws on the GPU:
//
//   PCG64 (XSL-RR 128/64, numpy's pcg64.h): state = state * M + inc, output
//   rotr(hi ^ lo, state >> 122); jump-ahead by Brown's O(log n) advance.
//   Ziggurat normal (numpy distributions.c random_standard_normal): 256
//   layers, tables copied from numpy (gf_ziggurat_tables.h); one draw per
//   normal on the fast path, extra draws on wedge / tail rejections.
//
// The sampler is sequential (a normal consumes a variable number of draws),
// so the stream is cut into segments of kSeg draws, one thread each:
//   K1 summary  walk the segment as if an attempt started at its first draw
//               (the "canonical" chain): normals produced, the overhang of
//               its last attempt into the next segment, and for the first
//               kWin positions the draws each attempt would consume and
//               whether it would yield.
//   K2 count    the true chain enters segment s at the previous segment's
//               overhang; within a few draws it lands on a canonical start
//               (chains re-synchronise on the first fast-path draw both
//               visit), so its count and its own overhang follow from K1.
//   K3 scan     exclusive prefix sum of the counts -> output index per segment.
//   K4 emit     regenerate the segment, walk the true chain, write
//               loc + scale * z to out[index] (numpy's random_normal).
// Every step rounds like the C code it restates (no FMA contraction).  The
// tail (|z| > 3.654, ~3e-4 of the draws) needs log1p exactly as the host
// libm rounds it (log1p_glibc below); the wedge test compares against exp,
// where a 1-ulp difference between CUDA and libm could only matter for a
// draw within 1 ulp of the layer boundary.  tests/test_gpu_generate.py
// checks the output against numpy bit for bit.

#include "gf_internal.h"
#include "gf_ziggurat_tables.h"

namespace gf {

using u128 = unsigned __int128;

__host__ __device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

struct Pcg {
  u128 s, inc;
};

__device__ __forceinline__ uint64_t pcg_next(Pcg& p) {
  p.s = p.s * pcg_mult() + p.inc;
  const uint64_t x = (uint64_t)(p.s >> 64) ^ (uint64_t)p.s;
  const unsigned r = (unsigned)(p.s >> 122);
  return (x >> r) | (x << ((64u - r) & 63u));
}

__device__ __forceinline__ double pcg_double(Pcg& p) {
  return __dmul_rn((double)(pcg_next(p) >> 11), 1.0 / 9007199254740992.0);
}

// state after `delta` more steps (Brown, "Random number generation with
// arbitrary strides", 1994 -- the advance numpy's pcg64_advance uses).
__device__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

// log1p as x86-64 glibc 2.39 computes it (numpy's npy_log1p calls libm):
// the fdlibm reduction with glibc's Estrin-form polynomial, built with FMA
// contraction in the polynomial sum and the k != 0 reconstruction (the
// ifunc variant chosen on FMA-capable hosts).  CUDA's own log1p differs in
// the last bit on ~0.05% of inputs, which would change tail normals; this
// restatement matched libm on 2.2e5 sampled inputs (tools/ notes in
// DESIGN.md).
__device__ double log1p_glibc(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double two54 = 1.80143985094819840000e+16;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int hx = __double2hiint(x);
  const int ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : __longlong_as_double(0x7ff8000000000000LL);
    if (ax < 0x3e200000) {
      if (__dadd_rn(two54, x) > 0.0 && ax < 0x3c900000) return x;
      return __dsub_rn(x, __dmul_rn(__dmul_rn(x, x), 0.5));
    }
    if (hx > 0 || hx <= (int)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return __dadd_rn(x, x);
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = __dadd_rn(1.0, x);
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double dk = (double)k;
  const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  if (hu == 0) {   // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = __dadd_rn(c, __dmul_rn(dk, ln2_lo));
      return __dadd_rn(__dmul_rn(dk, ln2_hi), c);
    }
    const double R = __dmul_rn(hfsq, __dsub_rn(1.0, __dmul_rn(0.66666666666666666, f)));
    if (k == 0) return __dsub_rn(f, R);
    return __dsub_rn(__dmul_rn(dk, ln2_hi), __dsub_rn(__dsub_rn(R, __dadd_rn(__dmul_rn(dk, ln2_lo), c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z4, z2);
  const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
  double R = __fma_rn(z, Lp1, __dmul_rn(z2, R2));
  R = __fma_rn(z4, R3, R);
  R = __fma_rn(z6, R4, R);
  const double sR = __dmul_rn(s, __dadd_rn(hfsq, R));
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, sR));
  const double inner = __dadd_rn(sR, __fma_rn(dk, ln2_lo, c));
  return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(hfsq, inner), f));
}

struct Attempt {
  int c;      // draws consumed (>= 1)
  int y;      // 1: yields a normal, 0: rejected (the next attempt follows), -1: runaway
  double v;
};

// One ziggurat attempt whose first draw is r; p is the generator just after
// r (taken by value: the extra draws are peeked, the caller's stream walks
// them itself).  numpy distributions.c random_standard_normal.
__device__ Attempt zig_attempt(uint64_t r, Pcg p) {
  Attempt a{1, 1, 0.0};
  const int idx = (int)(r & 0xff);
  r >>= 8;
  const uint64_t sign = r & 1;
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
  double x = __dmul_rn((double)rabs, kZigWi[idx]);
  if (sign) x = -x;
  if (rabs < kZigKi[idx]) {   // ~99.3%
    a.v = x;
    return a;
  }
  if (idx == 0) {             // tail beyond kZigR
    for (;;) {
      const double xx = __dmul_rn(-kZigInvR, log1p_glibc(-pcg_double(p)));
      const double yy = -log1p_glibc(-pcg_double(p));
      a.c += 2;
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
        const double t = __dadd_rn(kZigR, xx);
        a.v = ((rabs >> 8) & 1) ? -t : t;
        return a;
      }
      if (a.c > 201) {
        a.y = -1;
        return a;
      }
    }
  }
  const double u = pcg_double(p);
  a.c = 2;
  const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(kZigFi[idx - 1], kZigFi[idx]), u), kZigFi[idx]);
  if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
    a.v = x;
    return a;
  }
  a.y = 0;
  return a;
}

constexpr int kSeg = 1024;   // draws per segment (one thread)
constexpr int kWin = 64;     // re-synchronisation window at the segment head

struct SegSum {
  uint64_t ybits;      // position p < kWin: an attempt there would yield
  uint64_t cbits;      // position p < kWin: a start of the canonical chain
  uint32_t count;      // normals of the canonical chain
  uint32_t exit;       // overhang of its last attempt into the next segment
  uint8_t c[kWin];     // draws an attempt at p < kWin would consume (capped)
};

__device__ __forceinline__ Pcg seg_state(u128 base, u128 inc, int64_t seg) {
  return Pcg{pcg_advance(base, inc, (uint64_t)seg * kSeg), inc};
}

__global__ void zig_summary(u128 base, u128 inc, int64_t nseg, SegSum* __restrict__ out,
                            unsigned* __restrict__ err) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  Pcg p = seg_state(base, inc, s);
  SegSum r{};
  int next = 0;
  for (int pos = 0; pos < kSeg; ++pos) {
    const uint64_t d = pcg_next(p);
    const bool start = pos == next;
    if (pos < kWin || start) {
      const Attempt a = zig_attempt(d, p);
      if (a.y < 0) atomicOr(err, 1u);
      if (pos < kWin) {
        r.c[pos] = (uint8_t)min(a.c, 255);
        if (a.y > 0) r.ybits |= 1ULL << pos;
      }
      if (start) {
        next = pos + a.c;
        r.count += a.y > 0 ? 1u : 0u;
        if (pos < kWin) r.cbits |= 1ULL << pos;
      }
    }
  }
  r.exit = (uint32_t)(next - kSeg);
  if (r.exit >= kWin) atomicOr(err, 2u);
  out[s] = r;
}

// normals produced by the true chain of segment s (entering at the previous
// segment's overhang)
__global__ void zig_count(int64_t nseg, const SegSum* __restrict__ sum, uint32_t* __restrict__ count,
                          unsigned* __restrict__ err) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const SegSum& r = sum[s];
  int p = s == 0 ? 0 : (int)sum[s - 1].exit;
  uint32_t cnt = 0;
  while (p < kWin && !((r.cbits >> p) & 1)) {
    cnt += (uint32_t)((r.ybits >> p) & 1);
    p += r.c[p];
  }
  if (p >= kWin) {   // did not re-synchronise inside the window
    atomicOr(err, 4u);
    count[s] = 0;
    return;
  }
  const uint64_t before = p == 0 ? 0 : (r.ybits & r.cbits & ((1ULL << p) - 1));
  count[s] = cnt + r.count - (uint32_t)__popcll(before);
}

// exclusive prefix sums of 32-bit counts into 64-bit offsets: per-block scan,
// then a sequential pass over the block totals, then the block offsets
constexpr int kScanBlock = 1024;

__global__ void scan_blocks(const uint32_t* __restrict__ in, int64_t n, uint64_t* __restrict__ out,
                            uint64_t* __restrict__ block_tot) {
  __shared__ uint64_t sh[kScanBlock];
  const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const uint64_t v = i < n ? in[i] : 0;
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < kScanBlock; o <<= 1) {
    const uint64_t t = threadIdx.x >= (unsigned)o ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] += t;
    __syncthreads();
  }
  if (i < n) out[i] = sh[threadIdx.x] - v;
  if (threadIdx.x == kScanBlock - 1) block_tot[blockIdx.x] = sh[threadIdx.x];
}

__global__ void scan_totals(uint64_t* __restrict__ tot, int64_t nb, uint64_t* __restrict__ grand) {
  if (threadIdx.x != 0) return;
  uint64_t s = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const uint64_t t = tot[b];
    tot[b] = s;
    s += t;
  }
  *grand = s;
}

__global__ void scan_add(uint64_t* __restrict__ out, int64_t n, const uint64_t* __restrict__ tot) {
  const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  if (i < n) out[i] += tot[blockIdx.x];
}

// Normal j (C order over a virtual ncol-wide array) goes to
// out[(j / ncol) * rs + (j % ncol) * cs]: rs = ld, cs = 1 fills a padded
// row-major matrix; rs = 1, cs = ld its transpose.
template <typename T>
__global__ void zig_emit(u128 base, u128 inc, int64_t nseg, const SegSum* __restrict__ sum,
                         const uint64_t* __restrict__ offs, int64_t total, double loc, double scale,
                         T* __restrict__ out, int64_t ncol, int64_t rs, int64_t cs) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  uint64_t j = offs[s];
  if (j >= (uint64_t)total) return;
  int64_t r = (int64_t)(j / (uint64_t)ncol), c = (int64_t)(j % (uint64_t)ncol);
  Pcg p = seg_state(base, inc, s);
  int next = s == 0 ? 0 : (int)sum[s - 1].exit;
  for (int pos = 0; pos < kSeg; ++pos) {
    const uint64_t d = pcg_next(p);
    if (pos != next) continue;
    const Attempt a = zig_attempt(d, p);
    next = pos + a.c;
    if (a.y > 0) {
      if (j >= (uint64_t)total) return;
      out[r * rs + c * cs] = (T)__dadd_rn(loc, __dmul_rn(scale, a.v));   // random_normal: loc + scale * z
      ++j;
      if (++c == ncol) { c = 0; ++r; }
    }
  }
}

// A_ij <- s_i * (A_ij + t_i)  (the svm generator's label shift and sign flip,
// generators.py svm: lab * (A + lab / n))
__global__ void rows_affine_kernel(int64_t m, int64_t n, double* __restrict__ A, int64_t lda,
                                   const double* __restrict__ s, const double* __restrict__ t) {
  const int64_t total = m * n;
  for (int64_t k = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / n, j = k % n;
    double* a = A + i * lda + j;
    *a = __dmul_rn(s[i], __dadd_rn(*a, t[i]));
  }
}

void rows_affine(int64_t m, int64_t n, double* A, int64_t lda, const double* s, const double* t, cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  rows_affine_kernel<<<(unsigned)std::min<int64_t>(ceil_div(m * n, 256), 148 * 64), 256, 0, st>>>(m, n, A, lda, s, t);
  GF_CHECK_LAUNCH();
}

void normal_fill(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count,
                 double loc, double scale, int dtype, void* out, int64_t ncol, int64_t rs, int64_t cs,
                 cudaStream_t st) {
  if (count <= 0) return;
  const u128 base = ((u128)state_hi << 64) | state_lo;
  const u128 inc = ((u128)inc_hi << 64) | inc_lo;
  double margin = 1.03;
  for (int attempt = 0; attempt < 4; ++attempt, margin += 0.05) {
    const int64_t draws = (int64_t)((double)count * margin) + 4 * kWin;
    const int64_t nseg = ceil_div(draws, (int64_t)kSeg);
    const int64_t nb = ceil_div(nseg, (int64_t)kScanBlock);
    DBuf sums(nseg * sizeof(SegSum)), counts(nseg * sizeof(uint32_t)), offs(nseg * sizeof(uint64_t));
    DBuf tot((nb + 1) * sizeof(uint64_t)), err(sizeof(unsigned));
    GF_CUDA(cudaMemsetAsync(err.p, 0, sizeof(unsigned), st));
    const unsigned g = (unsigned)ceil_div(nseg, (int64_t)128);
    zig_summary<<<g, 128, 0, st>>>(base, inc, nseg, sums.as<SegSum>(), err.as<unsigned>());
    zig_count<<<g, 128, 0, st>>>(nseg, sums.as<SegSum>(), counts.as<uint32_t>(), err.as<unsigned>());
    scan_blocks<<<(unsigned)nb, kScanBlock, 0, st>>>(counts.as<uint32_t>(), nseg, offs.as<uint64_t>(),
                                                     tot.as<uint64_t>());
    scan_totals<<<1, 32, 0, st>>>(tot.as<uint64_t>(), nb, tot.as<uint64_t>() + nb);
    scan_add<<<(unsigned)nb, kScanBlock, 0, st>>>(offs.as<uint64_t>(), nseg, tot.as<uint64_t>());
    GF_CHECK_LAUNCH();
    uint64_t produced = 0;
    unsigned e = 0;
    GF_CUDA(cudaMemcpyAsync(&produced, tot.as<uint64_t>() + nb, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    GF_CUDA(cudaMemcpyAsync(&e, err.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    GF_CUDA(cudaStreamSynchronize(st));
    GF_REQUIRE(e == 0, GF_E_NUMERIC, "device normal sampler: ziggurat stream did not re-synchronise");
    if (produced < (uint64_t)count) continue;   // more draws needed than the margin allowed
    if (dtype == GF_F32)
      zig_emit<float><<<g, 128, 0, st>>>(base, inc, nseg, sums.as<SegSum>(), offs.as<uint64_t>(), count, loc,
                                          scale, (float*)out, ncol, rs, cs);
    else
      zig_emit<double><<<g, 128, 0, st>>>(base, inc, nseg, sums.as<SegSum>(), offs.as<uint64_t>(), count, loc,
                                           scale, (double*)out, ncol, rs, cs);
    GF_CHECK_LAUNCH();
    GF_CUDA(cudaStreamSynchronize(st));
    return;
  }
  GF_REQUIRE(false, GF_E_NUMERIC, "device normal sampler: draw budget exhausted");
}

}  // namespace gf
