// Internal object layouts and cross-file declarations of the C-ABI library.
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "gf_common.cuh"
#include "gf_terms.cuh"

// ------------------------------------------------------------- objects --
struct gf_matrix {
  int dtype = GF_F64;     // arithmetic type of the stored matrix
  int64_t m = 0, n = 0;   // logical shape (this rank's rows)
  int64_t ld = 0;         // padded row stride (elements)
  void* data = nullptr;   // device, m * ld elements
  size_t esize() const { return dtype == GF_F32 ? 4 : 8; }
};

struct gf_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

// true when collectives must run (a communicator exists, even of one rank)
inline bool comm_active(const gf_comm* c) { return c != nullptr && c->comm != nullptr; }

namespace gf {

// Stream of the API call in progress on this thread (set by the C entry
// points that take a stream): DBuf scratch buffers are allocated and freed
// in that stream's order, so a buffer released while kernels that use it are
// still queued (e.g. an early CGLS exit) cannot be handed out again before
// they ran -- also when the caller works on a non-blocking stream.
inline cudaStream_t& tls_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}
struct StreamScope {
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(tls_stream()) { tls_stream() = s; }
  ~StreamScope() { tls_stream() = prev; }
};

// Device buffer with RAII free, from the device's stream-ordered memory pool
// (cudaMallocAsync on the current call's stream; gf_init raises the pool's
// release threshold so freed blocks are reused instead of returned to the
// driver).  Plain cudaMalloc/cudaFree cost milliseconds and cudaFree
// synchronizes the device, which showed up as ~0.3 s per solve in the
// end-to-end path.  Buffers owned by long-lived handles are freed by the
// destroy calls (no stream: the legacy stream), after the API's result calls
// have synchronized the stream they were used on.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  explicit DBuf(size_t b) { alloc(b); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DBuf& operator=(DBuf&& o) noexcept { std::swap(p, o.p); std::swap(bytes, o.bytes); return *this; }
  ~DBuf() { if (p) cudaFreeAsync(p, tls_stream()); }
  void alloc(size_t b) {
    if (p) cudaFreeAsync(p, tls_stream());
    p = nullptr;
    bytes = b;
    if (b) {
      const auto t0 = std::chrono::steady_clock::now();
      GF_CUDA(cudaMallocAsync(&p, b, tls_stream()));
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ms > 2.0 && getenv("GF_VERBOSE_SETUP")) fprintf(stderr, "[gf] slow alloc %zu bytes: %.1f ms\n", b, ms);
    }
  }
  template <typename T> T* as() const { return (T*)p; }
};

// ------------------------------------------------ dense setup (gf_dense) --
// Gram scratch: bytes of the pre-split fp16 copy gram_tf32x3 can use for A
// (0 when the f16 pre-split path does not apply); `scratch` may be null.
size_t gram_scratch_bytes(const gf_matrix* A, bool tall);
void gram_accumulate(const gf_matrix* A, bool tall, double* G, int64_t ldg, cudaStream_t st,
                     void* scratch = nullptr, size_t scratch_bytes = 0, const unsigned* amax_known = nullptr);
void gram_tf32x3(const gf_matrix* A, double* G, int64_t ldg, cudaStream_t st, void* scratch = nullptr,
                 size_t scratch_bytes = 0, const unsigned* amax_known = nullptr);  // tcgen05, G += A'A
// fp64 tall Gram on the int8 tensor cores (exact int8 slices, gf_syrk_tc.cu);
// false when it does not apply (no scratch, GF_GRAM_F64=dmma)
bool gram_f64_i8(const gf_matrix* A, double* G, int64_t ldg, cudaStream_t st, void* scratch, size_t scratch_bytes);
void gram_finish(double* G, int64_t q, int64_t ldg, cudaStream_t st);
int cholesky(double* G, int64_t q, int64_t ld, int* d_info, cudaStream_t st);
void trtri(double* L, int64_t q, int64_t ld, double* tmp, cudaStream_t st);
void inverse_from_factor_inv(const double* W, int64_t q, int64_t ld, double* Ginv, cudaStream_t st);
void store_matrix(const double* src, int64_t lds, int dtype, void* dst, int64_t ldd, int64_t rows,
                  int64_t cols, cudaStream_t st);

// --------------------------------------------------- matrices (gf_matrix) --
void matrix_upload(gf_matrix* M, const void* src, int src_dtype, int64_t src_ld, cudaStream_t st);
void matrix_to_f64(const gf_matrix* M, double* dst_dev, cudaStream_t st);  // dense m x n
// amax (optional, zeroed by the caller): max |A_hat| over the real columns, as float bits
void scale_matrix(gf_matrix* M, const double* d, const double* e, cudaStream_t st, unsigned* amax = nullptr);
// y = A x (x: n) / y = A' x (x: m); fp64 device vectors; ws >= matvec_ws_bytes.
void matvec(const gf_matrix* A, bool transpose, const double* x, double* y, cudaStream_t st);
// y = (A o A) x / (A o A)' x (equilibration diagnostics, p = 2).
void sq_matvec(const gf_matrix* A, bool transpose, const double* x, double* y, cudaStream_t st);

// ---------------------------------------------- equilibration (gf_equil) --
struct EquilResult {
  int64_t sweeps;
  bool converged;
  double gamma;
  double fro2 = -1.0;   // ||D A E||_F^2 of the result (from the last column sums), -1 if not formed
};
// per-sweep observer (on_sweep of equilibration.py:178-179): sweep k, host
// copies of d_k^(1/2) (m) and e_k^(1/2) (n)
typedef void (*SweepCb)(int64_t k, const double* d, const double* e, int64_t m, int64_t n, void* user);
EquilResult equilibrate(gf_matrix* A, double gamma, double eps, int64_t max_iter, gf_comm* comm,
                        double* d_dev, double* e_dev, cudaStream_t st, SweepCb cb = nullptr, void* user = nullptr);
void rescale_even(gf_matrix* A, double* d_dev, double* e_dev, gf_comm* comm, cudaStream_t st);
// rescale_even with ||D A E||_F^2 already known (EquilResult::fro2): no pass over A
void rescale_even_fro2(gf_matrix* A, double* d_dev, double* e_dev, double fro2, gf_comm* comm, cudaStream_t st);

// --------------------------------------------------- vectors (gf_vec.cu) --
// Device copy of a gf_terms (h int8 + five fp64 arrays), owned.
struct TermsDev {
  DBuf buf;
  int64_t n = 0;
  TermsView view{};
  void load(const gf_terms* t, cudaStream_t st);
};
void prox_separable(const TermsView& t, int64_t n, const double* rho, const double* v, double* out,
                    cudaStream_t st);
void prox_base(int kind, int64_t n, const double* rho, const double* v, double* out, cudaStream_t st);
double evaluate(const TermsView& t, int64_t n, const double* v, cudaStream_t st);
void eval_base(int kind, int64_t n, const double* x, double* out, cudaStream_t st);
void conj_base(int kind, int64_t n, const double* w, double* out, cudaStream_t st);
double conjugate(const TermsView& t, int64_t n, const double* w, bool* supported, cudaStream_t st);
bool conj_supported(const TermsView& t, int64_t n, cudaStream_t st);
// true if any term's (effective) kind is one whose prox is an iterative
// Newton solve (NegEntr, Logistic): variable, up to 100-step epilogues
bool has_newton_prox(const TermsView& t, int64_t n, cudaStream_t st);

// ------------------------------------------------- CGLS indirect (gf_cgls) --
int64_t cgls_solve(const gf_matrix* A, bool tall, gf_comm* comm, const double* h1, const double* h2, double* z,
                   double tol, int64_t max_inner, bool* ok, cudaStream_t st);
int64_t project_indirect_dev(const gf_matrix* A, bool tall, gf_comm* comm, const double* c, const double* d,
                             const double* xw, const double* yw, double tol, int64_t max_inner, double* x,
                             double* y, bool* ok, cudaStream_t st);

// ------------------------------------------------- input synthesis (gf_rng) --
void normal_fill(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count,
                 double loc, double scale, int dtype, void* out, int64_t ncol, int64_t rs, int64_t cs,
                 cudaStream_t st);
void rows_affine(int64_t m, int64_t n, double* A, int64_t lda, const double* s, const double* t, cudaStream_t st);

// ------------------------------------------------------------- NCCL glue --
void allreduce_sum(gf_comm* c, double* buf, size_t count, cudaStream_t st);

// Pointer helpers: copy host-or-device fp64 arrays.
void copy_in(double* dst_dev, const double* src, int64_t n, cudaStream_t st);
void copy_out(double* dst, const double* src_dev, int64_t n, cudaStream_t st);

}  // namespace gf

struct gf_projector {
  gf_matrix* A = nullptr;   // not owned
  int mode = 0;             // 0 direct, 1 indirect
  bool tall = true;
  int64_t q = 0, ldq = 0;   // reduced dimension, padded stride of Ginv
  double tol = 1e-8;
  int64_t max_inner = 100;
  gf::DBuf gram;            // fp64 q x ldg (I + A'A or I + AA')
  int64_t ldg = 0;
  gf::DBuf ginv;            // working dtype, q x ldq: (I + A'A)^-1
  gf_comm* comm = nullptr;
};

struct gf_setup {
  gf_matrix* A = nullptr;   // owned: A_hat = D A E after creation
  gf::DBuf d, e;            // fp64 scalings (m local, n)
  gf_projector* P = nullptr;
  gf_setup_info info{};
  gf_comm* comm = nullptr;
};
