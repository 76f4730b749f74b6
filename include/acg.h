/*
 * acg.h — C ABI of the B200-native matrix-free PCG library (libacg_cuda.so).
 *
 * This is the drop-in boundary for the hot path of arXiv 1302.7193 ("anisocg"):
 * plain pointers and sizes, no C++ or torch types. The host C++ shim
 * (the headers under include/anisocg/) and the Python module (_anisocg) sit on top of it
 * with the reference's own names and signatures; each entry point below cites
 * the reference interface (under /root/reference/proj) it replaces.
 *
 * Conventions
 *  - Every function returns an acg_status; on failure acg_last_error() returns a
 *    thread-local message. ACG_ERR_INVALID_ARGUMENT maps to std::invalid_argument,
 *    ACG_ERR_BREAKDOWN to anisocg::NumericalBreakdown (operator.hpp:21-24).
 *  - Precision is fixed per context (ACG_F64 = double, ACG_F32 = float), like the
 *    template parameter T of OperatorContext<T> (operator.hpp:29-67).
 *  - Host field buffers use the reference's linear layouts (field.hpp:21-28):
 *      ACG_LAYOUT_VERTICAL   l = n_z*(m*i + j) + k   (numpy (m, m, n_z), C order)
 *      ACG_LAYOUT_HORIZONTAL l = m*(n_z*j + k) + i
 *    Device fields always use the library's own plane-major layout.
 *  - Scalars cross the ABI as double regardless of T (converted exactly like
 *    the reference's static_cast<double> pushes, solver.hpp:196-364).
 *  - Results are deterministic for a fixed slab count; for power-of-two slab
 *    counts dividing m they are bit-identical to the reference CPU code.
 */
#ifndef ACG_H
#define ACG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACG_ABI_VERSION 2

typedef enum {
    ACG_OK = 0,
    ACG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    ACG_ERR_BREAKDOWN = 2,        /* anisocg::NumericalBreakdown */
    ACG_ERR_CUDA = 3,
    ACG_ERR_NCCL = 4,
    ACG_ERR_INTERNAL = 5
} acg_status;

typedef enum { ACG_F64 = 0, ACG_F32 = 1 } acg_dtype;

/* field.hpp:21 Layout */
typedef enum { ACG_LAYOUT_VERTICAL = 0, ACG_LAYOUT_HORIZONTAL = 1 } acg_layout;

/* solver.hpp:16-17 */
typedef enum { ACG_VARIANT_STANDARD = 0, ACG_VARIANT_INTERLEAVED = 1 } acg_variant;
typedef enum { ACG_BACKEND_MATRIX_FREE = 0, ACG_BACKEND_CSR = 1 } acg_backend;

/* Arithmetic mode of the kernels.
 *  ACG_MATH_EXACT: IEEE round-to-nearest for every +,-,*,/ in the reference's
 *                  association order (no FMA contraction) — bit-identical to
 *                  the reference built with -ffp-contract=off.
 *  ACG_MATH_FAST:  FMA contraction and one reciprocal per Thomas level;
 *                  agrees with the reference to ~1e-15 relative per sweep. */
typedef enum { ACG_MATH_EXACT = 0, ACG_MATH_FAST = 1 } acg_math;

typedef struct acg_context acg_context; /* OperatorContext<T> on device slabs */
typedef struct acg_field acg_field;     /* Field3D<T> on device slabs */
typedef struct acg_comm acg_comm;       /* NCCL communicator (one rank per GPU) */
typedef struct acg_solver acg_solver;   /* device-resident PCG state (FusedState<T>) */

/* ------------------------------------------------------------------ basics */
const char* acg_last_error(void);
int acg_abi_version(void);
acg_status acg_device_count(int* count);
/* Pinned host buffers for fast host<->device copies (optional). */
acg_status acg_host_alloc(void** ptr, size_t bytes);
acg_status acg_host_free(void* ptr);

/* ------------------------------------------------------------- communicator
 * One process per GPU. rank 0 calls acg_comm_unique_id and distributes the
 * 128 bytes (e.g. via torch.distributed); every rank then calls
 * acg_comm_create. NCCL is loaded lazily (dlopen) only here. */
acg_status acg_comm_unique_id(void* id128);
acg_status acg_comm_create(acg_comm** out, int rank, int nranks, const void* id128, int device);
/* Peer-memory communicator for the ranks of ONE node (no NCCL): halo planes
 * and reduction slab sums are written straight into the neighbours' / peers'
 * device mailboxes through CUDA IPC mappings (NVLink P2P between GPUs; ranks
 * may also share a GPU) — in the interleaved loop by the sweep and reduction
 * kernels themselves — with completion signalled by release/acquire flags in
 * peer memory. `id128`: identical on all ranks, unique per communicator (16
 * random bytes broadcast by rank 0 are enough; the first 16 are used);
 * contexts must be created in the same order on every rank (their mailboxes
 * rendezvous under /dev/shm). */
acg_status acg_comm_create_ipc(acg_comm** out, int rank, int nranks, const void* id128,
                               int device);
acg_status acg_comm_destroy(acg_comm* comm);

/* ------------------------------------------------------------------ context
 * Replaces OperatorContext<T>(VerticalProfile, PanelGeometry), operator.hpp:32-44.
 * Arrays are the double-precision outputs of build_vertical_profile
 * (profile.hpp:18-26) and build_*_panel (grid.hpp:30-44), indexed exactly as there. */
typedef struct {
    int m;                    /* horizontal cells per panel side */
    int n_z;                  /* vertical levels */
    const double* a_prime;    /* n_z */
    const double* b_prime;    /* n_z */
    const double* c_prime;    /* n_z */
    const double* d;          /* n_z */
    const double* cell_area;  /* m*m, index i*m + j */
    const double* alpha_east; /* (m-1)*m, edge (i,j)-(i+1,j), index i*m + j */
    const double* alpha_north;/* m*(m-1), edge (i,j)-(i,j+1), index i*(m-1) + j */
    const double* alpha_diag; /* m*m */
} acg_operator_desc;

/* Where the panel lives. NULL placement = whole panel on the current device.
 * The panel is split into contiguous i-slabs (whole columns, paper Sec. 7).
 *  - comm == NULL, slabs = p >= 1: all p slabs on `device` in this process
 *    (halos by device copies) — the multi-GPU decomposition on one GPU;
 *  - comm != NULL: this rank owns slab `rank` of `nranks` on `device`. */
typedef struct {
    int device;
    int slabs;
    acg_comm* comm;
    acg_math math;
} acg_placement;

acg_status acg_context_create(acg_context** out, acg_dtype dtype, const acg_operator_desc* desc,
                              const acg_placement* placement);

/* The i-slab decomposition a context with p slabs uses (host only, no GPU):
 * slab s owns i-planes [i_begin[s], i_begin[s+1]); *exact_tree = 1 when the slabs
 * are nodes of the reference's pairwise reduction tree (parallel.hpp:11-20), so
 * the multi-slab reductions are bit-identical to the single-device ones. */
acg_status acg_partition_plan(int m, int p, int* i_begin /* p+1 */, int* exact_tree);
acg_status acg_context_destroy(acg_context* ctx);

typedef struct {
    int m, n_z, dtype, math;
    int nslabs_total;   /* p */
    int nslabs_local;   /* slabs owned by this process */
    int rank;           /* comm rank or 0 */
    int i_begin, i_end; /* i-range owned by this process */
    int exact_tree;     /* 1 if reductions reproduce the reference tree bit-for-bit */
    size_t bytes_per_field_local;
    int thomas_tmem;    /* 1 if the Thomas sweeps keep z' in TMEM with branch-free
                           divisions (their operand ranges validated at creation) */
} acg_context_info;
acg_status acg_context_info_get(const acg_context* ctx, acg_context_info* out);
acg_status acg_synchronize(const acg_context* ctx);

/* ------------------------------------------------------------------- fields
 * Replaces Field3D<T> storage (field.hpp:57-93). Host transfers take the
 * full m*m*n_z panel in `layout` (scope ACG_HOST_FULL, like the reference) or
 * only this process's i-range (ACG_HOST_LOCAL: (i_end-i_begin, m, n_z) in the
 * vertical layout, (m, n_z, i_end-i_begin) in the horizontal one). */
typedef enum { ACG_HOST_FULL = 0, ACG_HOST_LOCAL = 1 } acg_host_scope;

acg_status acg_field_create(acg_field** out, const acg_context* ctx);
acg_status acg_field_destroy(acg_field* f);
acg_status acg_field_upload(acg_field* f, const void* host, acg_layout layout, acg_host_scope scope);
acg_status acg_field_download(const acg_field* f, void* host, acg_layout layout, acg_host_scope scope);
/* Device-resident counterparts of upload/download: `dev` is a device buffer
 * (CUDA pointer, e.g. a torch/CuPy tensor's data) in the same host layout
 * convention; the relayout runs on the context's stream and the call returns
 * without synchronising (order later host work with acg_synchronize). */
acg_status acg_field_upload_device(acg_field* f, const void* dev, acg_layout layout,
                                   acg_host_scope scope);
acg_status acg_field_download_device(const acg_field* f, void* dev, acg_layout layout,
                                     acg_host_scope scope);
/* Asynchronous host transfers (no reference counterpart: the B200-side
 * overlap of PCIe traffic with the solver). The DMA and the relayout run on
 * the context's copy stream into the field's own staging, after the work
 * already enqueued on the context's stream; the call returns at once. The
 * host buffer must be page-locked (acg_host_alloc, cudaHostAlloc,
 * cudaHostRegister) and stay untouched until the transfer completes: every
 * later entry point that takes the field orders its device work after it, and
 * acg_field_wait blocks the host until it is done (required before reading a
 * downloaded buffer or reusing an uploaded one). */
acg_status acg_field_upload_async(acg_field* f, const void* host, acg_layout layout,
                                  acg_host_scope scope);
acg_status acg_field_download_async(const acg_field* f, void* host, acg_layout layout,
                                    acg_host_scope scope);
acg_status acg_field_wait(const acg_field* f);
acg_status acg_field_fill(acg_field* f, double value);
/* fill_random, field.hpp:180-196 (splitmix64, canonical (i,j,k) draw order) */
acg_status acg_field_fill_random(acg_field* f, uint64_t seed);
acg_status acg_field_copy(acg_field* dst, const acg_field* src);

/* --------------------------------------------------- operator and BLAS-1
 * apply            operator.hpp:101-135   y <- A x
 * precondition     operator.hpp:141-191   x <- M^-1 y
 * axpy/scal/dot/nrm2 field.hpp:116-173
 * true_residual    solver.hpp:61-69       ||f - A u||  (fused, one pass) */
acg_status acg_apply(const acg_context* ctx, const acg_field* x, acg_field* y);
acg_status acg_precondition(const acg_context* ctx, const acg_field* y, acg_field* x);
acg_status acg_axpy(double alpha, const acg_field* x, acg_field* y);
acg_status acg_scal(double alpha, acg_field* x);
acg_status acg_dot(const acg_field* x, const acg_field* y, double* out);
acg_status acg_nrm2(const acg_field* x, double* out);
acg_status acg_true_residual(const acg_context* ctx, const acg_field* u, const acg_field* f,
                             double* out);

/* ------------------------------------------------------ fused sweeps
 * interleaved_spmv_kernel operator.hpp:214-266: u += a p; p = z + b p;
 *                         q = A z + b q; returns sigma = <p, q>.
 * interleaved_prec_kernel operator.hpp:272-346: r -= a q; z = M^-1 r;
 *                         returns ||r|| and kappa = <r, z>. */
acg_status acg_interleaved_spmv_kernel(const acg_context* ctx, acg_field* u, acg_field* p,
                                       acg_field* q, const acg_field* z, double alpha,
                                       double beta, double* sigma);
acg_status acg_interleaved_prec_kernel(const acg_context* ctx, acg_field* r, acg_field* z,
                                       const acg_field* q, double alpha, double* r_norm,
                                       double* kappa);

/* ------------------------------------------------------------------ solver
 * SolverConfig / KernelTimings / SolveResult, solver.hpp:19-58. */
typedef struct {
    double epsilon;  /* relative tolerance, default 1e-5 */
    double tau;      /* absolute tolerance, default 1e-20 */
    int maxiter;     /* default 500 */
    int variant;     /* acg_variant */
    int backend;     /* acg_backend: MATRIX_FREE, or CSR = the reference's CsrBackend
                        (solver.hpp:126-145; standard variant only): stencil stored as CSR
                        plus stored tridiagonals, assembled on the device on first use */
    int workers;     /* accepted and ignored (OpenMP threads in the reference) */
    int record_timings; /* 1: per-kernel-family CUDA-event times in acg_solve_result */
    int layout;      /* acg_layout of the caller's fields; orders the CSR rows and entries
                        like assemble_csr(ctx, f.layout()) (csr.hpp:92-124), hence the
                        CSR summation order. acg_solve_host uses its layout argument. */
} acg_solver_config;

typedef struct { /* seconds, solver.hpp:39-47 */
    double spmv, prec, blas, fused_spmv, fused_prec, setup, total;
} acg_kernel_timings;

typedef struct {
    int iterations;
    int converged;
    double true_residual;
    int n_residual, n_kappa, n_alpha, n_beta; /* history lengths written */
    acg_kernel_timings timings;
    long long kernel_launches; /* device kernels launched by this solve */
    /* Library-allocated copies of the residual, kappa, alpha and beta histories
     * (n_residual, n_kappa, n_alpha, n_beta entries), filled for every history
     * whose caller buffer is NULL; free them with acg_solve_result_release.
     * This is how a caller with an "unbounded" maxiter (the reference only
     * pushes what runs, solver.hpp:196-364) gets histories without
     * pre-allocating maxiter+2 entries. */
    double* history[4];
} acg_solve_result;

void acg_solver_config_default(acg_solver_config* cfg);
/* Frees res->history[*] (safe on a zeroed or already released result). */
void acg_solve_result_release(acg_solve_result* res);

/* solve(), solver.hpp:373-378. Device fields; u0 may be NULL (zero start).
 * History buffers, when not NULL, need room for maxiter+2 doubles each; pass
 * NULL to receive library-allocated copies in res->history instead.
 * Concurrent calls on one context are safe: they serialise on the context. */
acg_status acg_solve(const acg_context* ctx, const acg_field* f, const acg_field* u0,
                     const acg_solver_config* cfg, acg_field* u_out, acg_solve_result* res,
                     double* residual_history, double* kappa_history, double* alpha_history,
                     double* beta_history);

/* Step-level control of the interleaved loop (device resident, asynchronous):
 * create -> start (init sweeps, solver.hpp:288-336) -> iterate(n) ... -> finish.
 * iterate() only enqueues work; iterations past convergence are no-ops. */
acg_status acg_solver_create(acg_solver** out, const acg_context* ctx, const acg_solver_config* cfg);
acg_status acg_solver_destroy(acg_solver* s);
acg_status acg_solver_start(acg_solver* s, const acg_field* f, const acg_field* u0);
acg_status acg_solver_iterate(acg_solver* s, int n);
acg_status acg_solver_finish(acg_solver* s, acg_field* u_out, acg_solve_result* res,
                             double* residual_history, double* kappa_history,
                             double* alpha_history, double* beta_history);
/* CUDA stream (cudaStream_t) the context's first local slab runs on. */
void* acg_context_stream(const acg_context* ctx);
/* Stream ordering with a caller's stream (cudaStream_t; NULL = the legacy
 * default stream), e.g. torch.cuda.current_stream(): the context's stream
 * waits for the work enqueued on `stream` so far (before reading a caller's
 * device buffer), or `stream` waits for the context's work (before the caller
 * consumes a result). Host-side non-blocking. */
acg_status acg_context_wait_stream(const acg_context* ctx, void* stream);
acg_status acg_stream_wait_context(void* stream, const acg_context* ctx);
/* Frees the context's cached scratch (solver work fields, scratch-field
 * pool, host-transfer staging); they are re-created on demand. */
acg_status acg_context_release_scratch(const acg_context* ctx);
/* Per-launch device time of the fused sweeps enqueued since the last call (ms,
 * CUDA events on the launching stream): returns counts and summed times. */
acg_status acg_solver_kernel_times(acg_solver* s, int* n_prec, double* ms_prec, int* n_spmv,
                                   double* ms_spmv);
/* Turn per-launch event timing of the fused sweeps on/off for iterate(). */
acg_status acg_solver_time_kernels(acg_solver* s, int enable);

/* ------------------------------------------------ host-buffer entry points
 * What the reference-facing shim calls: upload, run, download, in one call.
 * Buffers are full panels in `layout` (see above). */
acg_status acg_apply_host(const acg_context* ctx, acg_layout layout, const void* x, void* y);
acg_status acg_precondition_host(const acg_context* ctx, acg_layout layout, const void* y, void* x);
acg_status acg_true_residual_host(const acg_context* ctx, acg_layout layout, const void* u,
                                  const void* f, double* out);
acg_status acg_solve_host(const acg_context* ctx, acg_layout layout, const void* f,
                          const void* u0, const acg_solver_config* cfg, void* u_out,
                          acg_solve_result* res, double* residual_history,
                          double* kappa_history, double* alpha_history, double* beta_history);

/* Kernel launches issued by this process so far (all entry points). */
long long acg_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* ACG_H */
