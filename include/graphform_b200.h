/*
 * graphform_b200.h -- C ABI of the B200-native POGS graph-form ADMM hot path.
 *
 * The reference (`graphform`, pure Python) has no FFI; its path sits behind
 * Python functions.  Each entry point below replaces one of them -- the
 * citation is the reference function it stands in for (paths relative to
 * /root/reference/pkg/src/graphform/).  The Python host layer
 * (paper_1503_08366_b200/_native.py) binds these with ctypes and maps the
 * GF_E_* codes onto the reference exception classes (errors.py:4-25).
 *
 * Conventions
 *  - Plain C types only.  Vector arguments are fp64 and may be host or device
 *    pointers (CUDA UVA; copies use cudaMemcpyDefault) unless marked DEVICE.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *    Calls are stream-ordered and return after their outputs are written
 *    (they synchronize the stream when they hand results to the host).
 *  - Matrices live in library-owned device memory, row-major, row stride
 *    padded to 128 bytes (zero padding).  dtype is GF_F32 or GF_F64: the
 *    arithmetic type of the matrix passes (GEMV, Gram).  Term math, norms and
 *    the stopping rule are always fp64.
 *  - Every call returns GF_OK or a GF_E_* code; gf_last_error() gives the
 *    message of the last failure on the calling thread.
 */
#ifndef GRAPHFORM_B200_H_
#define GRAPHFORM_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GF_OK 0
#define GF_E_DIMENSION 1        /* errors.py:8  DimensionError        */
#define GF_E_PARAMETER 2        /* errors.py:12 ParameterError        */
#define GF_E_DEGENERATE_INPUT 3 /* errors.py:16 DegenerateInputError  */
#define GF_E_NUMERIC 4          /* errors.py:20 NumericError          */
#define GF_E_CUDA 5
#define GF_E_NCCL 6
#define GF_E_UNSUPPORTED 7

#define GF_F32 0
#define GF_F64 1

/* solver status codes (solver.py:46-49) */
#define GF_STATUS_RUNNING 0
#define GF_STATUS_SOLVED 1
#define GF_STATUS_MAX_ITERATIONS 2
#define GF_STATUS_DEGENERATE 3

typedef struct gf_matrix gf_matrix;
typedef struct gf_projector gf_projector;
typedef struct gf_setup gf_setup;
typedef struct gf_solver gf_solver;
typedef struct gf_comm gf_comm;

/* Separable function as flat term arrays c*h(a*x-b)+d*x+(e/2)x^2
 * (functions.py:193-225).  h holds the BaseFunction codes 0..9 (enum order,
 * functions.py:34-60) narrowed to int8. */
typedef struct {
  int64_t n;
  const int8_t* h;
  const double* a;
  const double* b;
  const double* c;
  const double* d;
  const double* e;
} gf_terms;

/* SolverSettings (solver.py:52-92); projection: 0 direct, 1 indirect. */
typedef struct {
  double rho0, abs_tol, rel_tol;
  int64_t max_iter;
  double alpha;
  int adaptive_rho;
  double delta, tau;
  int projection;
  double projection_tol; /* <= 0: the decreasing schedule (solver.py:398-406) */
  int gap_stop;          /* solver.py:378-390: also stop on the duality gap at the
                            full iterate (problem.py:67-85) */
} gf_settings;

/* Per-iteration scalars handed to callbacks (solver.py:359-360) and the
 * final result fields of SolveResult (solver.py:95-109). */
typedef struct {
  int status;
  int64_t iterations;      /* SolveResult.iterations                    */
  int64_t k;               /* index of the last recorded iteration, -1 if none */
  double r_pri, r_dual, eps_pri, eps_dual;
  double rho;              /* rho of iteration k (callback argument)    */
  double objective;
  double final_rho;        /* SolveResult.final_rho                     */
  int64_t inner_iterations;/* CGLS inner iterations of iteration k      */
  double gap;              /* SolveResult.gap of the last gap test       */
  int gap_valid;           /* 0: no gap (gap_stop off or a conjugate unsupported) */
} gf_solver_state;

typedef struct {
  int64_t sweeps;          /* Equilibration.iterations */
  int converged;
  double gamma;
  double setup_seconds;    /* device time of prepare() */
} gf_setup_info;

/* ------------------------------------------------------------ runtime -- */
const char* gf_version(void);
const char* gf_last_error(void);
int gf_init(int device); /* select device; idempotent */

/* ----------------------------------------------------- prox / evaluate -- */
/* prox.py:113-138 prox_separable: out_i = prox of term i at rho_i, v_i.
 * All pointers DEVICE, length t->n; rho must be positive and finite. */
int gf_prox_separable(const gf_terms* t, const double* rho, const double* v,
                      double* out, void* stream);
/* prox.py:101-110 prox_base: one base kind, elementwise (DEVICE pointers). */
int gf_prox_base(int64_t n, int kind, const double* rho, const double* v,
                 double* out, void* stream);
/* functions.py:307-327 SeparableFunction.evaluate -> *result (host). */
int gf_evaluate(const gf_terms* t, const double* v, double* result, void* stream);
/* functions.py:160-164 eval_base, elementwise (DEVICE pointers). */
int gf_eval_base(int64_t n, int kind, const double* x, double* out, void* stream);
/* functions.py:147-150 conjugate_base: h*(w) elementwise (DEVICE pointers). */
int gf_conj_base(int64_t n, int kind, const double* w, double* out, void* stream);
/* functions.py:329-365 SeparableFunction.conjugate: sum_i f_i*(w_i) -> *result
 * (host); *supported = 0 when some term has e > 0 and a kind without a closed
 * form (the reference returns None).  Term and w pointers DEVICE. */
int gf_conjugate(const gf_terms* t, const double* w, double* result, int* supported, void* stream);

/* ------------------------------------------------------------ matrices -- */
/* problem.py:30-49 (coercion of A): copy an m x n row-major matrix
 * (host or device, src_dtype GF_F32/GF_F64, leading dimension src_ld) into
 * library memory as `dtype`.  Host sources are staged through pinned memory. */
int gf_matrix_create(int dtype, int64_t m, int64_t n, const void* src, int src_dtype,
                     int64_t src_ld, void* stream, gf_matrix** out);
int gf_matrix_destroy(gf_matrix* A);
int gf_matrix_shape(const gf_matrix* A, int64_t* m, int64_t* n, int64_t* ld, int* dtype);
/* copy the (possibly scaled) matrix back as fp64 m x n row-major (tests). */
int gf_matrix_download(const gf_matrix* A, double* dst, void* stream);
/* y = A x (x: n, y: m) and y = A' x (x: m, y: n), fp64 vectors; the matvecs
 * behind residual_stop (solver.py:197-198) and the CGLS handles. */
int gf_matvec(const gf_matrix* A, int transpose, const double* x, double* y, void* stream);
/* y = (A o A) x and y = (A o A)' x (elementwise squares, fp64 vectors, host or
 * device): the p = 2 |A|^p matvec handles of equilibration.py:94-125 that
 * check_equilibrated (:227-267) and equilibration_objective (:270-287) use. */
int gf_sq_matvec(const gf_matrix* A, int transpose, const double* x, double* y, void* stream);

/* ------------------------------------------------------- equilibration -- */
/* equilibration.py:134-197 equilibrate: regularised Sinkhorn-Knopp, p = 2.
 * gamma < 0 / eps <= 0 select the reference defaults.  d (m), e (n) receive
 * the square roots of the Sinkhorn iterates.  comm may be NULL (single GPU);
 * with a communicator A holds this rank's rows and the column sums are
 * all-reduced every sweep. */
int gf_equilibrate(gf_matrix* A, double gamma, double eps, int64_t max_iter,
                   gf_comm* comm, double* d, double* e, int64_t* sweeps,
                   int* converged, double* gamma_used, void* stream);
/* The same with the reference's on_sweep(k, d, e) observer
 * (equilibration.py:178-179): after each sweep's updates and before its
 * convergence test, on_sweep receives host copies of d_k^(1/2) (m values)
 * and e_k^(1/2) (n values).  on_sweep may be NULL. */
typedef void (*gf_sweep_fn)(int64_t k, const double* d, const double* e, int64_t m, int64_t n, void* user);
int gf_equilibrate_observed(gf_matrix* A, double gamma, double eps, int64_t max_iter,
                            gf_comm* comm, double* d, double* e, int64_t* sweeps,
                            int* converged, double* gamma_used, gf_sweep_fn on_sweep,
                            void* user, void* stream);
/* equilibration.py:214-224 rescale_even (in place on d, e). */
int gf_rescale_even(gf_matrix* A, double* d, double* e, gf_comm* comm, void* stream);
/* solver.py:142-145 _scale_matrix: A <- diag(d) A diag(e), in place. */
int gf_scale_matrix(gf_matrix* A, const double* d, const double* e, void* stream);

/* ---------------------------------------------------------- projection -- */
/* projection.py:61-99 build_projector.  mode 0 (direct): forms the Gram
 * I + A'A (m >= n) or I + AA' (m < n), factors it (blocked Cholesky, fp64)
 * and stores the inverse for the per-iteration apply; mode 1 (indirect):
 * CGLS only.  The projector references A (which must outlive it).
 * With a communicator (row partition) the Gram is all-reduced. */
int gf_projector_create(gf_matrix* A, int mode, double tol, int64_t max_inner,
                        gf_comm* comm, void* stream, gf_projector** out);
int gf_projector_destroy(gf_projector* P);
/* reduced Gram matrix (q x q fp64, host or device) -- ProjectorCache.gram */
int gf_projector_gram(const gf_projector* P, double* out, void* stream);
/* projection.py:112-127 project: (x, y) = Pi(c, d). */
int gf_project(gf_projector* P, const double* c, const double* d, double* x,
               double* y, void* stream);
/* projection.py:130-162 project_indirect (CGLS, warm start optional). */
int gf_project_indirect(gf_projector* P, const double* c, const double* d,
                        const double* x_warm, const double* y_warm, double tol,
                        double* x, double* y, int64_t* iterations, int* converged,
                        void* stream);

/* --------------------------------------------------------------- setup -- */
/* solver.py:148-169 prepare: equilibrate (equil != 0, unless d_in/e_in
 * given) + rescale_even + scale A in place + build the projector.
 * Takes ownership of A. */
int gf_setup_create(gf_matrix* A, int equil, const double* d_in, const double* e_in,
                    int mode, double tol, int64_t max_inner, gf_comm* comm,
                    void* stream, gf_setup** out);
int gf_setup_destroy(gf_setup* S);
int gf_setup_get_info(const gf_setup* S, gf_setup_info* info);
int gf_setup_scaling(const gf_setup* S, double* d, double* e, void* stream);
int gf_setup_projector(gf_setup* S, gf_projector** P);
int gf_setup_matrix(gf_setup* S, gf_matrix** A);

/* -------------------------------------------------------------- solver -- */
/* solver.py:248-437 solve, split into create / run / read so callbacks and
 * traces can observe every iteration.  f has this rank's m rows, g all n.
 * x0 (n) and nu0 (m) may be NULL (cold start). */
int gf_solver_create(gf_setup* S, const gf_terms* f, const gf_terms* g,
                     const gf_settings* settings, const double* x0, const double* nu0,
                     void* stream, gf_solver** out);
/* Run until the solve terminates or `steps` more iterations are recorded
 * (steps <= 0: to termination).  Iterations are launched in chunks with a
 * device-side stop rule; *st is the state after the last recorded one. */
int gf_solver_run(gf_solver* s, int64_t steps, gf_solver_state* st, void* stream);
/* per-iteration history rows (r_pri, r_dual, eps_pri, eps_dual, rho, obj)
 * for iterations [0, count) -> out (count x 6, host). */
int gf_solver_history(gf_solver* s, int64_t count, double* out, void* stream);
/* hat-space iterate of the last recorded iteration (IterationSnapshot,
 * solver.py:123-139): state that entered its prox and its half iterate. */
int gf_solver_snapshot(gf_solver* s, double* x_hat, double* y_hat, double* xt,
                       double* yt, double* x_half_hat, double* y_half_hat, void* stream);
/* SolveResult vectors (original variables): x, mu (n); y, nu (m). */
int gf_solver_result(gf_solver* s, double* x, double* y, double* mu, double* nu,
                     gf_solver_state* st, void* stream);
int gf_solver_destroy(gf_solver* s);
/* One-shot solve (the proposed gf_solve of SURVEY §8b): create, run to
 * termination, read SolveResult vectors (x, mu: n; y, nu: m; host or device)
 * and, if history != NULL, the per-iteration rows (r_pri, r_dual, eps_pri,
 * eps_dual, rho, objective) of iterations [0, st->k] into history
 * ((settings->max_iter + 1) x 6 doubles, host), then destroy. */
int gf_solve(gf_setup* S, const gf_terms* f, const gf_terms* g, const gf_settings* settings,
             const double* x0, const double* nu0, double* x, double* y, double* mu, double* nu,
             gf_solver_state* st, double* history, void* stream);
/* device time (ms) spent in solver iterations so far (CUDA events) */
int gf_solver_elapsed_ms(gf_solver* s, double* ms);
/* instrumentation: kernels launched so far; with profiling enabled, summed
 * CUDA-event durations and counts per kernel class (8 slots: 0 Ginv GEMV +
 * x side, 1 row pass + y side, 2 column pass, 3 slab reduce, 4 y scalars,
 * 5 Z step / controller, 6 all-reduce, 7 fused row + column pass). */
int gf_solver_stats(gf_solver* s, int64_t* launches, double* kernel_ms, int64_t* kernel_count);
int gf_solver_profile(gf_solver* s, int enable);

/* ------------------------------------------- input synthesis (§8f item 1) -- */
/* numpy Generator(PCG64).normal(loc, scale, size=count) -- the streams of the
 * reference generators (generators.py:80-264) -- bit for bit on the device.
 * (state, inc) is the generator's bit_generator.state (128-bit halves).
 * Normal j is written to out[(j / ncol) * rs + (j % ncol) * cs] as dtype
 * (GF_F32 rounds the fp64 value).  out is DEVICE memory. */
int gf_normal_fill(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count,
                   double loc, double scale, int dtype, void* out, int64_t ncol, int64_t rs, int64_t cs,
                   void* stream);
/* y = A x / y = A' x over a raw DEVICE matrix (m x n, row stride lda elements,
 * 16-byte aligned rows), fp64 accumulation; x, y DEVICE fp64.  The generators'
 * A @ v and A.T @ b. */
int gf_dense_matvec(int dtype, int64_t m, int64_t n, const void* A, int64_t lda, int transpose,
                    const double* x, double* y, void* stream);
/* A_ij <- s_i * (A_ij + t_i) on a DEVICE fp64 matrix (svm generator). */
int gf_rows_affine(int64_t m, int64_t n, double* A, int64_t lda, const double* s, const double* t, void* stream);
/* *all_finite <- 1 if every entry of the DEVICE matrix (dtype, m x n, row
 * stride lda) is finite, else 0: one read of A (the reference's
 * GraphFormProblem check "A must be finite", problem.py:35-49). */
int gf_matrix_all_finite(int dtype, int64_t m, int64_t n, const void* A, int64_t lda, int* all_finite,
                         void* stream);
/* dst (dtype, row stride ldd) <- src (fp64, row stride lds), DEVICE. */
int gf_convert_matrix(int64_t m, int64_t n, const double* src, int64_t lds, int dtype, void* dst, int64_t ldd,
                      void* stream);

/* ----------------------------------------------- multi-GPU (row shards) -- */
/* NCCL communicator for one process per GPU; the 128-byte unique id is made
 * by rank 0 and broadcast by the caller (torch.distributed in the host). */
int gf_comm_unique_id(char* id128);
int gf_comm_create(const char* id128, int nranks, int rank, gf_comm** out);
int gf_comm_destroy(gf_comm* c);

#ifdef __cplusplus
}
#endif
#endif /* GRAPHFORM_B200_H_ */
