// C-ABI entry points (include/graphform_b200.h): argument checks, object
// lifetimes, error-code mapping, projector/setup orchestration and NCCL glue.

#include <dlfcn.h>

#include <chrono>
#include <mutex>
#include <cstring>

#include "gf_internal.h"
#include "gf_gemv.cuh"

// implemented in gf_solver.cu
gf_solver* solver_create(gf_setup* S, const gf_terms* f, const gf_terms* g, const gf_settings* st_in,
                         const double* x0, const double* nu0, cudaStream_t st);
void solver_run(gf_solver* s, int64_t steps, gf_solver_state* out, cudaStream_t st);
void solver_history(gf_solver* s, int64_t count, double* out, cudaStream_t st);
void solver_snapshot(gf_solver* s, double* x_hat, double* y_hat, double* xt, double* yt, double* xhh, double* yhh,
                     cudaStream_t st);
void solver_result(gf_solver* s, double* x, double* y, double* mu, double* nu, gf_solver_state* out,
                   cudaStream_t st);
double solver_elapsed(gf_solver* s);
void solver_stats(gf_solver* s, int64_t* launches, double* kernel_ms, int64_t* kernel_count);
void solver_profile(gf_solver* s, int enable);
void solver_free(gf_solver* s);

namespace gf {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }
void throw_error(int code, const std::string& msg) { throw Error{code, msg}; }

int num_sms() {
  static thread_local int dev = -1, sms = 0;
  int d = 0;
  cudaGetDevice(&d);
  if (d != dev) {
    GF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d));
    dev = d;
  }
  return sms;
}

// NCCL is resolved at run time (dlopen), not linked: a process that loads this
// library before torch must not pin the system libnccl.so.2 (2.27) under the
// soname torch's own 2.28 copy needs.  An already-loaded libnccl.so.2 (torch's,
// whenever torch.distributed set up the ranks) is used first.
struct NcclApi {
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  const char* (*GetErrorString)(ncclResult_t);
};

static const NcclApi& nccl() {
  static std::mutex mu;
  static NcclApi api{};
  static bool ready = false;
  std::lock_guard<std::mutex> lk(mu);
  if (!ready) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) throw_error(GF_E_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* name) {
      void* f = dlsym(h, name);
      if (f == nullptr) throw_error(GF_E_NCCL, std::string("libnccl.so.2 lacks ") + name);
      return f;
    };
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    ready = true;
  }
  return api;
}

void allreduce_sum(gf_comm* c, double* buf, size_t count, cudaStream_t st) {
  if (!comm_active(c) || count == 0) return;
  const ncclResult_t r = nccl().AllReduce(buf, buf, count, ncclDouble, ncclSum, c->comm, st);
  if (r != ncclSuccess) throw_error(GF_E_NCCL, std::string("ncclAllReduce: ") + nccl().GetErrorString(r));
}

// Grow-only per-device scratch (from the retained pool, kept for the process) for
// large setup temporaries; a ScratchLock holds the device's arena for the
// duration of one projector build.
struct ScratchArena {
  std::mutex mu;
  void* p[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t bytes[4] = {0, 0, 0, 0};
};
static ScratchArena& arena_for_current_device() {
  static ScratchArena arenas[64];
  int dev = 0;
  GF_CUDA(cudaGetDevice(&dev));
  return arenas[dev & 63];
}
struct ScratchLock {
  ScratchArena& a;
  std::lock_guard<std::mutex> lk;
  ScratchLock() : a(arena_for_current_device()), lk(a.mu) {}
  void* get(int i, size_t bytes) {   // slot i, grown to at least `bytes`
    if (a.bytes[i] < bytes) {
      // from the stream-ordered pool, whose reserve gf_init pre-maps: a plain
      // cudaMalloc of the Gram's 4 GB pre-split copy cost ~0.3 s on first use
      if (a.p[i]) GF_CUDA(cudaFreeAsync(a.p[i], 0));
      a.p[i] = nullptr;
      a.bytes[i] = 0;
      GF_CUDA(cudaMallocAsync(&a.p[i], bytes, 0));
      GF_CUDA(cudaStreamSynchronize(0));
      a.bytes[i] = bytes;
    }
    return a.p[i];
  }
};
struct DBufView {
  void* p;
  explicit DBufView(void* q) : p(q) {}
  template <typename T> T* as() const { return (T*)p; }
};

// Setup phase timing (CUDA events), printed to stderr when GF_VERBOSE_SETUP=1.
struct PhaseTimer {
  cudaStream_t st;
  bool on;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  std::vector<double> host_ms;   // host clock at each mark (enqueue time)
  explicit PhaseTimer(cudaStream_t s) : st(s) {
    const char* e = getenv("GF_VERBOSE_SETUP");
    on = e && e[0] == '1';
    if (on) mark("start");
  }
  void mark(const char* name) {
    if (!on) return;
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, st);
    marks.emplace_back(name, ev);
    host_ms.push_back(std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now().time_since_epoch()).count());
  }
  void report(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    fprintf(stderr, "[gf] %s:", what);
    for (size_t i = 1; i < marks.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second);
      fprintf(stderr, " %s %.2f ms (host %.2f)", marks[i].first.c_str(), ms, host_ms[i] - host_ms[i - 1]);
    }
    fprintf(stderr, "\n");
  }
  ~PhaseTimer() {
    for (auto& m : marks) cudaEventDestroy(m.second);
  }
};

template <typename F>
static int guarded(F&& fn) {
  try {
    fn();
    return GF_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return GF_E_CUDA;
  }
}

template <typename F>
static int guarded(void* stream, F&& fn) {
  StreamScope scope((cudaStream_t)stream);
  return guarded(std::forward<F>(fn));
}

static bool host_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return !(at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
}

// fp64 vector argument that may live on the host: device view (copied if needed).
struct DevVec {
  const double* p = nullptr;
  DBuf own;
  DevVec(const double* src, int64_t n, cudaStream_t st) {
    if (src == nullptr || n <= 0) { p = src; return; }
    if (host_ptr(src)) {
      own.alloc(n * sizeof(double));
      copy_in(own.as<double>(), src, n, st);
      p = own.as<double>();
    } else {
      p = src;
    }
  }
};

__global__ void combine_kernel(const double* a, double sa, const double* b, double sb, double* out, int64_t n) {
  for (int64_t j = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    out[j] = sa * a[j] + sb * b[j];
}
static void combine(const double* a, double sa, const double* b, double sb, double* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  combine_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, st>>>(a, sa, b, sb, out, n);
  GF_CHECK_LAUNCH();
}

static void check_terms(const gf_terms* t) {
  GF_REQUIRE(t != nullptr, GF_E_PARAMETER, "terms must not be NULL");
  GF_REQUIRE(t->n >= 0, GF_E_DIMENSION, "negative length");
  GF_REQUIRE(t->n == 0 || (t->h && t->a && t->b && t->c && t->d && t->e), GF_E_PARAMETER, "null term array");
}

// lower triangle of a q x q row-major matrix (row stride ld) <-> packed rows
// (row i: i + 1 entries at i (i + 1) / 2); unpack = 1 writes it back
__global__ void lower_pack_kernel(double* __restrict__ G, int64_t q, int64_t ld, double* __restrict__ packed,
                                  int unpack) {
  const int64_t np = q * (q + 1) / 2;
  for (int64_t t = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; t < np; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (i * (i + 1) / 2 > t) --i;
    while ((i + 1) * (i + 2) / 2 <= t) ++i;
    const int64_t j = t - i * (i + 1) / 2;
    if (unpack) G[i * ld + j] = packed[t];
    else packed[t] = G[i * ld + j];
  }
}

static gf_projector* projector_build(gf_matrix* A, int mode, double tol, int64_t max_inner, gf_comm* comm,
                                     cudaStream_t st, const unsigned* amax_known = nullptr) {
  GF_REQUIRE(mode == 0 || mode == 1, GF_E_PARAMETER, "unknown projection mode");
  GF_REQUIRE(tol > 0.0, GF_E_PARAMETER, "projection tolerance must be positive");
  std::unique_ptr<gf_projector> P(new gf_projector());
  P->A = A;
  P->mode = mode;
  P->comm = comm;
  P->tall = A->m >= A->n;   // projection.py:76 (global rows decide under a partition)
  if (comm_active(comm)) {
    DBuf b(sizeof(double));
    double mloc = (double)A->m;
    GF_CUDA(cudaMemcpyAsync(b.p, &mloc, sizeof(double), cudaMemcpyHostToDevice, st));
    allreduce_sum(comm, b.as<double>(), 1, st);
    double mg = 0;
    GF_CUDA(cudaMemcpyAsync(&mg, b.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    GF_CUDA(cudaStreamSynchronize(st));
    P->tall = mg >= (double)A->n;
    GF_REQUIRE(P->tall, GF_E_UNSUPPORTED, "row-partitioned solves require a tall matrix");
  }
  P->q = P->tall ? A->n : A->m;
  P->tol = tol;
  P->max_inner = max_inner > 0 ? max_inner : std::max<int64_t>(100, 2 * std::min(A->m, A->n));
  if (mode == 1) return P.release();
  const int64_t q = P->q;
  P->ldg = padded_ld(q, GF_F64);
  P->ldq = padded_ld(q, A->dtype);
  const size_t gbytes = (size_t)std::max<int64_t>(q, 1) * P->ldg * sizeof(double);
  P->gram.alloc(gbytes);
  GF_CUDA(cudaMemsetAsync(P->gram.p, 0, gbytes, st));
  PhaseTimer pt(st);
  // large temporaries come from a grow-only per-device arena: growing the
  // stream-ordered pool by hundreds of MB mid-setup was measured to stall the
  // host for 10-250 ms on some boxes (slot 3: the Gram's pre-split copy of A,
  // used when it fits -- or already fits -- with 1 GB to spare)
  ScratchLock sl;
  void* gscratch = nullptr;
  size_t gsb = A->m > 0 && A->n > 0 ? gram_scratch_bytes(A, P->tall) : 0;
  if (gsb > 0 && sl.a.bytes[3] < gsb) {
    size_t free_b = 0, total_b = 0;
    GF_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (gsb - sl.a.bytes[3] + (1ull << 30) >= free_b) gsb = 0;
  }
  if (gsb > 0) gscratch = sl.get(3, gsb);
  if (A->m > 0 && A->n > 0) gram_accumulate(A, P->tall, P->gram.as<double>(), P->ldg, st, gscratch, gsb, amax_known);
  if (comm_active(comm)) {
    // the lower triangle is what every Gram path leaves valid (gram_finish
    // mirrors it): ship it packed, q (q + 1) / 2 doubles instead of q x ldg
    const size_t np = (size_t)q * (q + 1) / 2;
    DBuf packed(std::max<size_t>(np, 1) * sizeof(double));
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div((int64_t)np, 256), (int64_t)num_sms() * 8);
    lower_pack_kernel<<<g, 256, 0, st>>>(P->gram.as<double>(), q, P->ldg, packed.as<double>(), 0);
    GF_CHECK_LAUNCH();
    allreduce_sum(comm, packed.as<double>(), np, st);
    lower_pack_kernel<<<g, 256, 0, st>>>(P->gram.as<double>(), q, P->ldg, packed.as<double>(), 1);
    GF_CHECK_LAUNCH();
    GF_CUDA(cudaStreamSynchronize(st));   // `packed` is freed on scope exit
  }
  gram_finish(P->gram.as<double>(), q, P->ldg, st);
  pt.mark("gram");
  // q x q fp64 temporaries: the factor L (arena slot 0) and one buffer that
  // is first TRTRI's scratch and then, once W = L^-1 is formed in place, the
  // W'W output.  For an fp64 matrix that buffer is G^-1 itself (same padded
  // stride): 9.6 GB instead of 16 GB of q x q buffers at C3's q = 20000, so
  // a first build stays inside the pool's pre-mapped reserve.
  const bool direct = A->dtype == GF_F64 && P->ldq == P->ldg;
  if (direct) P->ginv.alloc(gbytes);
  DBufView L(sl.get(0, gbytes)), tmp(direct ? P->ginv.p : sl.get(1, gbytes));
  DBufView& inv = tmp;
  DBuf info(sizeof(int));
  GF_CUDA(cudaMemcpyAsync(L.p, P->gram.p, gbytes, cudaMemcpyDeviceToDevice, st));
  const int bad = cholesky(L.as<double>(), q, P->ldg, info.as<int>(), st);
  if (bad != 0)
    throw_error(GF_E_NUMERIC, "Gram factorization failed: leading minor of order " + std::to_string(bad) +
                                  " is not positive definite");
  pt.mark("cholesky");
  GF_CUDA(cudaMemsetAsync(tmp.p, 0, gbytes, st));
  trtri(L.as<double>(), q, P->ldg, tmp.as<double>(), st);
  pt.mark("trtri");
  inverse_from_factor_inv(L.as<double>(), q, P->ldg, inv.as<double>(), st);
  if (!direct) {
    P->ginv.alloc((size_t)std::max<int64_t>(q, 1) * P->ldq * A->esize());
    store_matrix(inv.as<double>(), P->ldg, A->dtype, P->ginv.p, P->ldq, q, q, st);
  }
  pt.mark("inverse");
  GF_CUDA(cudaStreamSynchronize(st));
  pt.report("projector_build");
  return P.release();
}

static void ginv_apply(gf_projector* P, const double* rhs, double* out, cudaStream_t st) {
  gf_matrix G;
  G.dtype = P->A->dtype;
  G.m = P->q; G.n = P->q; G.ld = P->ldq; G.data = P->ginv.p;
  matvec(&G, false, rhs, out, st);
}

static void project_direct(gf_projector* P, const double* c, const double* d, double* x, double* y, cudaStream_t st) {
  gf_matrix* A = P->A;
  const int64_t m = A->m, n = A->n;
  if (P->tall) {
    DBuf t(std::max<int64_t>(n, 1) * sizeof(double)), rhs(std::max<int64_t>(n, 1) * sizeof(double));
    GF_CUDA(cudaMemsetAsync(t.p, 0, t.bytes, st));
    if (m > 0) matvec(A, true, d, t.as<double>(), st);                 // A' d
    if (comm_active(P->comm)) allreduce_sum(P->comm, t.as<double>(), n, st);
    combine(c, 1.0, t.as<double>(), 1.0, rhs.as<double>(), n, st);     // c + A' d
    ginv_apply(P, rhs.as<double>(), x, st);                            // x = G^-1 (c + A' d)
    if (m > 0) matvec(A, false, x, y, st);                             // y = A x
  } else {
    DBuf t(std::max<int64_t>(m, 1) * sizeof(double)), w(std::max<int64_t>(m, 1) * sizeof(double));
    DBuf u(std::max<int64_t>(n, 1) * sizeof(double));
    matvec(A, false, c, t.as<double>(), st);                           // A c
    combine(t.as<double>(), 1.0, d, -1.0, t.as<double>(), m, st);      // A c - d
    ginv_apply(P, t.as<double>(), w.as<double>(), st);                 // w
    combine(d, 1.0, w.as<double>(), 1.0, y, m, st);                    // y = d + w
    matvec(A, true, w.as<double>(), u.as<double>(), st);
    combine(c, 1.0, u.as<double>(), -1.0, x, n, st);                   // x = c - A' w
  }
  GF_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gf

using namespace gf;

struct gf_solver;
namespace gf {
// one pass over A: any non-finite entry clears *ok (grid-stride over rows,
// lanes over columns; no temporaries)
template <typename T>
__global__ void all_finite_kernel(const T* __restrict__ A, int64_t m, int64_t n, int64_t lda, int* __restrict__ ok) {
  bool good = true;
  for (int64_t r = blockIdx.x; r < m; r += gridDim.x)
    for (int64_t c = threadIdx.x; c < n; c += blockDim.x) good &= isfinite(A[r * lda + c]);
  if (!__syncthreads_and(good) && threadIdx.x == 0) atomicExch(ok, 0);
}
}  // namespace gf

extern "C" {

const char* gf_version(void) { return "graphform-b200 0.1.0 (sm_100a)"; }
const char* gf_last_error(void) { return gf::last_error(); }

int gf_init(int device) {
  return guarded([&] {
    GF_CUDA(cudaSetDevice(device));
    GF_CUDA(cudaFree(0));
    num_sms();
    cudaMemPool_t pool;
    GF_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;   // retain freed blocks for reuse (DBuf)
    GF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    // Pre-map part of the pool once: growing it during a setup (hundreds of
    // MB at a time) was measured to stall the host for 10-150 ms per call.
    // GF_POOL_RESERVE_MB (default 12288; 0 disables) is kept mapped and reused.
    const char* env = getenv("GF_POOL_RESERVE_MB");
    const size_t mb = env ? (size_t)atoll(env) : (size_t)12288;
    if (mb > 0) {
      size_t free_b = 0, total_b = 0;
      GF_CUDA(cudaMemGetInfo(&free_b, &total_b));
      const size_t want = std::min(mb << 20, free_b / 4);
      void* p = nullptr;
      if (want > 0 && cudaMallocAsync(&p, want, 0) == cudaSuccess) {
        cudaFreeAsync(p, 0);
        GF_CUDA(cudaStreamSynchronize(0));
      } else {
        cudaGetLastError();
      }
    }
  });
}

int gf_prox_separable(const gf_terms* t, const double* rho, const double* v, double* out, void* stream) {
  return guarded(stream, [&] {
    check_terms(t);
    TermsView view{t->h, t->a, t->b, t->c, t->d, t->e};
    prox_separable(view, t->n, rho, v, out, (cudaStream_t)stream);
    GF_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  });
}

int gf_prox_base(int64_t n, int kind, const double* rho, const double* v, double* out, void* stream) {
  return guarded(stream, [&] {
    GF_REQUIRE(kind >= 0 && kind <= 9, GF_E_PARAMETER, "unknown base function code");
    prox_base(kind, n, rho, v, out, (cudaStream_t)stream);
    GF_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  });
}

int gf_evaluate(const gf_terms* t, const double* v, double* result, void* stream) {
  return guarded(stream, [&] {
    check_terms(t);
    TermsView view{t->h, t->a, t->b, t->c, t->d, t->e};
    *result = evaluate(view, t->n, v, (cudaStream_t)stream);
  });
}

int gf_eval_base(int64_t n, int kind, const double* x, double* out, void* stream) {
  return guarded(stream, [&] {
    GF_REQUIRE(kind >= 0 && kind <= 9, GF_E_PARAMETER, "unknown base function code");
    eval_base(kind, n, x, out, (cudaStream_t)stream);
    GF_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  });
}

int gf_normal_fill(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count,
                   double loc, double scale, int dtype, void* out, int64_t ncol, int64_t rs, int64_t cs,
                   void* stream) {
  return guarded(stream, [&] {
    GF_REQUIRE(dtype == GF_F32 || dtype == GF_F64, GF_E_PARAMETER, "dtype must be GF_F32 or GF_F64");
    GF_REQUIRE(count >= 0 && ncol >= 1, GF_E_DIMENSION, "count must be >= 0 and ncol >= 1");
    normal_fill(state_hi, state_lo, inc_hi, inc_lo, count, loc, scale, dtype, out, ncol, rs, cs,
                (cudaStream_t)stream);
  });
}

int gf_dense_matvec(int dtype, int64_t m, int64_t n, const void* A, int64_t lda, int transpose, const double* x,
                    double* y, void* stream) {
  return guarded(stream, [&] {
    GF_REQUIRE(dtype == GF_F32 || dtype == GF_F64, GF_E_PARAMETER, "dtype must be GF_F32 or GF_F64");
    const int64_t es = dtype == GF_F32 ? 4 : 8;
    GF_REQUIRE(m >= 0 && n >= 0 && lda >= n, GF_E_DIMENSION, "bad matrix shape / row stride");
    GF_REQUIRE(((uintptr_t)A % 16) == 0 && (lda * es) % 16 == 0, GF_E_PARAMETER,
               "matrix rows must be 16-byte aligned");
    gf_matrix view;
    view.dtype = dtype; view.m = m; view.n = n; view.ld = lda; view.data = const_cast<void*>(A);
    if (m == 0 || n == 0) {
      GF_CUDA(cudaMemsetAsync(y, 0, (transpose ? n : m) * sizeof(double), (cudaStream_t)stream));
      GF_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
      return;
    }
    matvec(&view, transpose != 0, x, y, (cudaStream_t)stream);
  });
}

int gf_rows_affine(int64_t m, int64_t n, double* A, int64_t lda, const double* s, const double* t, void* stream) {
  return guarded(stream, [&] {
    rows_affine(m, n, A, lda, s, t, (cudaStream_t)stream);
    GF_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  });
}

int gf_matrix_all_finite(int dtype, int64_t m, int64_t n, const void* A, int64_t lda, int* all_finite, void* stream) {
  return guarded(stream, [&] {
    GF_REQUIRE(dtype == GF_F32 || dtype == GF_F64, GF_E_PARAMETER, "dtype must be GF_F32 or GF_F64");
    cudaStream_t st = (cudaStream_t)stream;
    DBuf flag(sizeof(int));
    const int one = 1;
    GF_CUDA(cudaMemcpyAsync(flag.p, &one, sizeof(int), cudaMemcpyHostToDevice, st));
    if (m > 0 && n > 0) {
      const unsigned g = (unsigned)std::min<int64_t>(m, (int64_t)num_sms() * 16);
      if (dtype == GF_F32) all_finite_kernel<float><<<g, 256, 0, st>>>((const float*)A, m, n, lda, flag.as<int>());
      else all_finite_kernel<double><<<g, 256, 0, st>>>((const double*)A, m, n, lda, flag.as<int>());
      GF_CHECK_LAUNCH();
    }
    GF_CUDA(cudaMemcpyAsync(all_finite, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    GF_CUDA(cudaStreamSynchronize(st));
  });
}

int gf_convert_matrix(int64_t m, int64_t n, const double* src, int64_t lds, int dtype, void* dst, int64_t ldd,
                      void* stream) {
  return guarded(stream, [&] {
    GF_REQUIRE(dtype == GF_F32 || dtype == GF_F64, GF_E_PARAMETER, "dtype must be GF_F32 or GF_F64");
    store_matrix(src, lds, dtype, dst, ldd, m, n, (cudaStream_t)stream);
    GF_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  });
}

int gf_conj_base(int64_t n, int kind, const double* w, double* out, void* stream) {
  return guarded(stream, [&] {
    GF_REQUIRE(kind >= 0 && kind <= 9, GF_E_PARAMETER, "unknown base function code");
    conj_base(kind, n, w, out, (cudaStream_t)stream);
    GF_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  });
}

int gf_conjugate(const gf_terms* t, const double* w, double* result, int* supported, void* stream) {
  return guarded(stream, [&] {
    check_terms(t);
    TermsView view{t->h, t->a, t->b, t->c, t->d, t->e};
    bool ok = true;
    *result = conjugate(view, t->n, w, &ok, (cudaStream_t)stream);
    *supported = ok ? 1 : 0;
  });
}

int gf_matrix_create(int dtype, int64_t m, int64_t n, const void* src, int src_dtype, int64_t src_ld, void* stream,
                     gf_matrix** out) {
  return guarded(stream, [&] {
    GF_REQUIRE(dtype == GF_F32 || dtype == GF_F64, GF_E_PARAMETER, "dtype must be GF_F32 or GF_F64");
    GF_REQUIRE(src_dtype == GF_F32 || src_dtype == GF_F64, GF_E_PARAMETER, "bad source dtype");
    GF_REQUIRE(m >= 0 && n >= 1, GF_E_DIMENSION, "matrix must have at least one column");
    GF_REQUIRE(src != nullptr || m == 0, GF_E_PARAMETER, "null matrix");
    GF_REQUIRE(src_ld >= n, GF_E_DIMENSION, "leading dimension smaller than n");
    std::unique_ptr<gf_matrix> M(new gf_matrix());
    M->dtype = dtype;
    M->m = m;
    M->n = n;
    M->ld = padded_ld(n, dtype);
    const size_t bytes = (size_t)std::max<int64_t>(m, 1) * M->ld * M->esize();
    // from the stream-ordered pool (retained across solves): a plain
    // cudaMalloc/cudaFree of gigabytes maps/unmaps memory and was measured to
    // stall solve() teardown for up to 0.7 s
    GF_CUDA(cudaMallocAsync(&M->data, bytes, 0));
    if (m > 0) matrix_upload(M.get(), src, src_dtype, src_ld, (cudaStream_t)stream);
    GF_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    *out = M.release();
  });
}

int gf_matrix_destroy(gf_matrix* A) {
  return guarded([&] {
    if (A == nullptr) return;
    if (A->data) cudaFreeAsync(A->data, 0);
    delete A;
  });
}

int gf_matrix_shape(const gf_matrix* A, int64_t* m, int64_t* n, int64_t* ld, int* dtype) {
  return guarded([&] {
    if (m) *m = A->m;
    if (n) *n = A->n;
    if (ld) *ld = A->ld;
    if (dtype) *dtype = A->dtype;
  });
}

int gf_matrix_download(const gf_matrix* A, double* dst, void* stream) {
  return guarded(stream, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    if (A->m == 0) return;
    DBuf tmp((size_t)A->m * A->n * sizeof(double));
    matrix_to_f64(A, tmp.as<double>(), st);
    GF_CUDA(cudaMemcpyAsync(dst, tmp.p, (size_t)A->m * A->n * 8, cudaMemcpyDefault, st));
    GF_CUDA(cudaStreamSynchronize(st));
  });
}

int gf_matvec(const gf_matrix* A, int transpose, const double* x, double* y, void* stream) {
  return guarded(stream, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nx = transpose ? A->m : A->n, ny = transpose ? A->n : A->m;
    DevVec xv(x, nx, st);
    const bool yhost = ny > 0 && host_ptr(y);
    DBuf yb;
    double* yd = y;
    if (yhost) { yb.alloc(ny * sizeof(double)); yd = yb.as<double>(); }
    if (ny > 0 && nx > 0) matvec(A, transpose != 0, xv.p, yd, st);
    if (yhost) copy_out(y, yd, ny, st);
    GF_CUDA(cudaStreamSynchronize(st));
  });
}

int gf_sq_matvec(const gf_matrix* A, int transpose, const double* x, double* y, void* stream) {
  return guarded(stream, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nx = transpose ? A->m : A->n, ny = transpose ? A->n : A->m;
    DevVec xv(x, nx, st);
    const bool yhost = ny > 0 && host_ptr(y);
    DBuf yb;
    double* yd = y;
    if (yhost) { yb.alloc(ny * sizeof(double)); yd = yb.as<double>(); }
    if (ny > 0 && nx > 0) sq_matvec(A, transpose != 0, xv.p, yd, st);
    else if (ny > 0) GF_CUDA(cudaMemsetAsync(yd, 0, ny * sizeof(double), st));
    if (yhost) copy_out(y, yd, ny, st);
    GF_CUDA(cudaStreamSynchronize(st));
  });
}

int gf_equilibrate_observed(gf_matrix* A, double gamma, double eps, int64_t max_iter, gf_comm* comm, double* d, double* e,
                   int64_t* sweeps, int* converged, double* gamma_used, gf_sweep_fn on_sweep, void* user,
                            void* stream) {
  return guarded(stream, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    DBuf dd(std::max<int64_t>(A->m, 1) * sizeof(double)), ee(A->n * sizeof(double));
    const EquilResult r = equilibrate(A, gamma, eps, max_iter, comm, dd.as<double>(), ee.as<double>(), st,
                                      (SweepCb)on_sweep, user);
    copy_out(d, dd.as<double>(), A->m, st);
    copy_out(e, ee.as<double>(), A->n, st);
    GF_CUDA(cudaStreamSynchronize(st));
    if (sweeps) *sweeps = r.sweeps;
    if (converged) *converged = r.converged ? 1 : 0;
    if (gamma_used) *gamma_used = r.gamma;
  });
}
int gf_equilibrate(gf_matrix* A, double gamma, double eps, int64_t max_iter, gf_comm* comm, double* d, double* e,
                   int64_t* sweeps, int* converged, double* gamma_used, void* stream) {
  return gf_equilibrate_observed(A, gamma, eps, max_iter, comm, d, e, sweeps, converged, gamma_used, nullptr, nullptr,
                                 stream);
}


int gf_rescale_even(gf_matrix* A, double* d, double* e, gf_comm* comm, void* stream) {
  return guarded(stream, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    DBuf dd(std::max<int64_t>(A->m, 1) * sizeof(double)), ee(A->n * sizeof(double));
    copy_in(dd.as<double>(), d, A->m, st);
    copy_in(ee.as<double>(), e, A->n, st);
    rescale_even(A, dd.as<double>(), ee.as<double>(), comm, st);
    copy_out(d, dd.as<double>(), A->m, st);
    copy_out(e, ee.as<double>(), A->n, st);
    GF_CUDA(cudaStreamSynchronize(st));
  });
}

int gf_scale_matrix(gf_matrix* A, const double* d, const double* e, void* stream) {
  return guarded(stream, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    DevVec dv(d, A->m, st), ev(e, A->n, st);
    scale_matrix(A, dv.p, ev.p, st);
    GF_CUDA(cudaStreamSynchronize(st));
  });
}

int gf_projector_create(gf_matrix* A, int mode, double tol, int64_t max_inner, gf_comm* comm, void* stream,
                        gf_projector** out) {
  return guarded(stream, [&] { *out = projector_build(A, mode, tol, max_inner, comm, (cudaStream_t)stream); });
}

int gf_projector_destroy(gf_projector* P) {
  return guarded([&] { delete P; });
}

int gf_projector_gram(const gf_projector* P, double* out, void* stream) {
  return guarded(stream, [&] {
    GF_REQUIRE(P->mode == 0, GF_E_PARAMETER, "indirect projectors have no Gram matrix");
    cudaStream_t st = (cudaStream_t)stream;
    GF_CUDA(cudaMemcpy2DAsync(out, P->q * sizeof(double), P->gram.p, P->ldg * sizeof(double), P->q * sizeof(double),
                              P->q, cudaMemcpyDefault, st));
    GF_CUDA(cudaStreamSynchronize(st));
  });
}

int gf_project(gf_projector* P, const double* c, const double* d, double* x, double* y, void* stream) {
  return guarded(stream, [&] {
    GF_REQUIRE(P->mode == 0, GF_E_PARAMETER, "project requires a direct-mode cache; use project_indirect");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t m = P->A->m, n = P->A->n;
    DevVec cv(c, n, st), dv(d, m, st);
    DBuf xb(std::max<int64_t>(n, 1) * sizeof(double)), yb(std::max<int64_t>(m, 1) * sizeof(double));
    project_direct(P, cv.p, dv.p, xb.as<double>(), yb.as<double>(), st);
    copy_out(x, xb.as<double>(), n, st);
    copy_out(y, yb.as<double>(), m, st);
    GF_CUDA(cudaStreamSynchronize(st));
  });
}

int gf_project_indirect(gf_projector* P, const double* c, const double* d, const double* x_warm,
                        const double* y_warm, double tol, double* x, double* y, int64_t* iterations, int* converged,
                        void* stream) {
  return guarded(stream, [&] {
    GF_REQUIRE(tol > 0.0, GF_E_PARAMETER, "projection tolerance must be positive");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t m = P->A->m, n = P->A->n;
    DevVec cv(c, n, st), dv(d, m, st), xw(x_warm, n, st), yw(y_warm, m, st);
    DBuf xb(std::max<int64_t>(n, 1) * sizeof(double)), yb(std::max<int64_t>(m, 1) * sizeof(double));
    bool ok = false;
    const int64_t it = project_indirect_dev(P->A, P->tall, P->comm, cv.p, dv.p, x_warm ? xw.p : nullptr,
                                            y_warm ? yw.p : nullptr, tol, P->max_inner, xb.as<double>(),
                                            yb.as<double>(), &ok, st);
    copy_out(x, xb.as<double>(), n, st);
    copy_out(y, yb.as<double>(), m, st);
    GF_CUDA(cudaStreamSynchronize(st));
    if (iterations) *iterations = it;
    if (converged) *converged = ok ? 1 : 0;
  });
}

int gf_setup_create(gf_matrix* A, int equil, const double* d_in, const double* e_in, int mode, double tol,
                    int64_t max_inner, gf_comm* comm, void* stream, gf_setup** out) {
  return guarded(stream, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    const auto t0 = std::chrono::steady_clock::now();
    std::unique_ptr<gf_setup> S(new gf_setup());
    S->comm = comm;
    S->d.alloc(std::max<int64_t>(A->m, 1) * sizeof(double));
    S->e.alloc(A->n * sizeof(double));
    S->info.sweeps = 0;
    S->info.converged = 1;
    S->info.gamma = 0.0;
    if (d_in != nullptr && e_in != nullptr) {
      copy_in(S->d.as<double>(), d_in, A->m, st);
      copy_in(S->e.as<double>(), e_in, A->n, st);
    } else if (equil) {
      PhaseTimer pt(st);
      const EquilResult r = equilibrate(A, -1.0, -1.0, 300, comm, S->d.as<double>(), S->e.as<double>(), st);
      pt.mark("equilibrate");
      // the Frobenius norm comes from the last sweep's column sums (no pass
      // over A; GF_RESCALE_PASS=1 forms it with rescale_even's row pass)
      static const bool pass = [] {
        const char* ev = getenv("GF_RESCALE_PASS");
        return ev && ev[0] == '1';
      }();
      if (r.fro2 >= 0.0 && !pass) rescale_even_fro2(A, S->d.as<double>(), S->e.as<double>(), r.fro2, comm, st);
      else rescale_even(A, S->d.as<double>(), S->e.as<double>(), comm, st);
      pt.mark("rescale");
      pt.report("setup");
      S->info.sweeps = r.sweeps;
      S->info.converged = r.converged ? 1 : 0;
      S->info.gamma = r.gamma;
    } else {
      std::vector<double> ones(std::max(A->m, A->n), 1.0);
      copy_in(S->d.as<double>(), ones.data(), A->m, st);
      copy_in(S->e.as<double>(), ones.data(), A->n, st);
    }
    DBuf amax(sizeof(unsigned));   // max |A_hat| for the Gram's fp16 split, from the scaling pass
    GF_CUDA(cudaMemsetAsync(amax.p, 0, sizeof(unsigned), st));
    scale_matrix(A, S->d.as<double>(), S->e.as<double>(), st, amax.as<unsigned>());
    S->P = projector_build(A, mode, tol, max_inner, comm, st, amax.as<unsigned>());
    S->A = A;  // ownership transferred on success only
    GF_CUDA(cudaStreamSynchronize(st));
    S->info.setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = S.release();
  });
}

int gf_setup_destroy(gf_setup* S) {
  return guarded([&] {
    if (!S) return;
    delete S->P;
    if (S->A) gf_matrix_destroy(S->A);
    delete S;
  });
}

int gf_setup_get_info(const gf_setup* S, gf_setup_info* info) {
  return guarded([&] { *info = S->info; });
}

int gf_setup_scaling(const gf_setup* S, double* d, double* e, void* stream) {
  return guarded(stream, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    if (d) copy_out(d, S->d.as<double>(), S->A->m, st);
    if (e) copy_out(e, S->e.as<double>(), S->A->n, st);
    GF_CUDA(cudaStreamSynchronize(st));
  });
}

int gf_setup_projector(gf_setup* S, gf_projector** P) {
  return guarded([&] { *P = S->P; });
}

int gf_setup_matrix(gf_setup* S, gf_matrix** A) {
  return guarded([&] { *A = S->A; });
}

int gf_solver_create(gf_setup* S, const gf_terms* f, const gf_terms* g, const gf_settings* settings,
                     const double* x0, const double* nu0, void* stream, gf_solver** out) {
  return guarded(stream, [&] {
    check_terms(f);
    check_terms(g);
    GF_REQUIRE(settings->max_iter >= 1, GF_E_PARAMETER, "max_iter must be at least 1");
    *out = solver_create(S, f, g, settings, x0, nu0, (cudaStream_t)stream);
  });
}

int gf_solver_run(gf_solver* s, int64_t steps, gf_solver_state* st, void* stream) {
  return guarded(stream, [&] { solver_run(s, steps, st, (cudaStream_t)stream); });
}

int gf_solver_history(gf_solver* s, int64_t count, double* out, void* stream) {
  return guarded(stream, [&] { solver_history(s, count, out, (cudaStream_t)stream); });
}

int gf_solver_snapshot(gf_solver* s, double* x_hat, double* y_hat, double* xt, double* yt, double* x_half_hat,
                       double* y_half_hat, void* stream) {
  return guarded(stream, [&] { solver_snapshot(s, x_hat, y_hat, xt, yt, x_half_hat, y_half_hat, (cudaStream_t)stream); });
}

int gf_solver_result(gf_solver* s, double* x, double* y, double* mu, double* nu, gf_solver_state* st, void* stream) {
  return guarded(stream, [&] { solver_result(s, x, y, mu, nu, st, (cudaStream_t)stream); });
}

int gf_solver_destroy(gf_solver* s) {
  return guarded([&] { solver_free(s); });
}

int gf_solve(gf_setup* S, const gf_terms* f, const gf_terms* g, const gf_settings* settings, const double* x0,
             const double* nu0, double* x, double* y, double* mu, double* nu, gf_solver_state* st,
             double* history, void* stream) {
  return guarded(stream, [&] {
    check_terms(f);
    check_terms(g);
    GF_REQUIRE(settings->max_iter >= 1, GF_E_PARAMETER, "max_iter must be at least 1");
    const cudaStream_t cs = (cudaStream_t)stream;
    struct Owner {
      gf_solver* p = nullptr;
      ~Owner() { if (p) solver_free(p); }
    } s;
    s.p = solver_create(S, f, g, settings, x0, nu0, cs);
    gf_solver_state tmp{};
    gf_solver_state* out = st ? st : &tmp;
    solver_run(s.p, 0, out, cs);
    solver_result(s.p, x, y, mu, nu, out, cs);
    if (history != nullptr && out->k >= 0) solver_history(s.p, out->k + 1, history, cs);
  });
}

int gf_solver_elapsed_ms(gf_solver* s, double* ms) {
  return guarded([&] { *ms = solver_elapsed(s); });
}

int gf_solver_stats(gf_solver* s, int64_t* launches, double* kernel_ms, int64_t* kernel_count) {
  return guarded([&] { solver_stats(s, launches, kernel_ms, kernel_count); });
}

int gf_solver_profile(gf_solver* s, int enable) {
  return guarded([&] { solver_profile(s, enable); });
}

int gf_comm_unique_id(char* id128) {
  return guarded([&] {
    ncclUniqueId id;
    const ncclResult_t r = nccl().GetUniqueId(&id);
    if (r != ncclSuccess) throw_error(GF_E_NCCL, std::string("ncclGetUniqueId: ") + nccl().GetErrorString(r));
    std::memcpy(id128, id.internal, sizeof(id.internal));
  });
}

int gf_comm_create(const char* id128, int nranks, int rank, gf_comm** out) {
  return guarded([&] {
    GF_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, GF_E_PARAMETER, "bad rank / world size");
    std::unique_ptr<gf_comm> c(new gf_comm());
    c->nranks = nranks;
    c->rank = rank;
    {   // a communicator even for one rank, so every collective call site is exercisable on one GPU
      ncclUniqueId id;
      std::memcpy(id.internal, id128, sizeof(id.internal));
      const ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, id, rank);
      if (r != ncclSuccess) throw_error(GF_E_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
    }
    *out = c.release();
  });
}

int gf_comm_destroy(gf_comm* c) {
  return guarded([&] {
    if (!c) return;
    if (c->comm) nccl().CommDestroy(c->comm);
    delete c;
  });
}

}  // extern "C"
