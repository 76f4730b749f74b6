// Internal types shared by the kernels (acg_kernels.cu) and the runtime
// (acg_runtime.cu). Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <atomic>

#include <cstddef>
#include <cstdint>

namespace acg {

// Device field layout ("plane-major"): a slab owning global
// i-planes [i0, i0 + m_loc) stores element (i, j, k) at
//     (i - i0) * plane + k * m + j,      plane = n_z * m,
// so a warp of 32 consecutive j is one coalesced 256 B (fp64) row, the vertical
// neighbour is +-m and the i-neighbour is +-plane. One ghost plane precedes
// plane 0 and one follows plane m_loc-1; they receive the neighbouring slabs'
// boundary planes (halo exchange). Contiguous i-slabs keep each slab's column
// partials a contiguous block of the reference's column order col = i*m + j.

// Rows of the per-slab profile table (n_z entries each), converted to T on the
// host exactly like OperatorContext<T> (operator.hpp:36-43).
enum ProfRow { kProfS = 0,   // (a'_k - b'_k) - c'_k   (operator.hpp:127, :307)
               kProfB = 1,   // b'_k
               kProfC = 2,   // c'_k
               kProfD = 3,   // d_k
               kProfInvD = 4,// 1 / d_k          (fast math only)
               kProfRows = 5 };

// Rows of the per-slab column table (m_loc * m entries each, index il*m + j).
enum ColRow { kColArea = 0,  // |T|
              kColDiag = 1,  // alpha_diag
              kColAtil = 2,  // alpha_diag / |T| in T (operator.hpp:163, :302)
              kColE = 3,     // alpha toward i+1 (0 on the panel edge), operator.hpp:81
              kColW = 4,     // alpha toward i-1
              kColN = 5,     // alpha toward j+1
              kColS = 6,     // alpha toward j-1
              kColInvA = 7,  // 1 / |T|          (fast math only)
              kColRows = 8 };

// Peer-memory halo fused into the interleaved sweeps (IPC transport, ranks > 1,
// DESIGN.md §6). Producer (K1, k_thomas_tm): the CTAs of plane 0 / plane m_loc-1
// also store their z columns into the neighbour's mailbox slot and the last CTA
// of the plane releases the neighbour's flag. Consumer (K2, k_fused_spmv_pair2):
// the CTAs of the boundary planes acquire the flag and read the ghost rows from
// this rank's mailbox. Side 0 = toward rank r-1 (plane 0 / ghost plane -1),
// side 1 = toward rank r+1 (plane m_loc-1 / ghost plane m_loc).
template <typename T>
struct HaloLink {
    T* put[2] = {nullptr, nullptr};                        // neighbour's mailbox slot
    unsigned long long* put_flag[2] = {nullptr, nullptr};  // neighbour's flag
    unsigned* arrive = nullptr;                            // [2] CTA arrivals (zero at rest)
    const T* ghost[2] = {nullptr, nullptr};                // own mailbox slots
    const unsigned long long* wait_flag[2] = {nullptr, nullptr};
    unsigned long long seq = 0;
    int on = 0;
};

template <typename T>
struct SlabView {
    int m, n_z, m_loc, i0;
    long long plane;  // n_z * m
    const T* prof;    // kProfRows x n_z
    const T* col;     // kColRows x (m_loc * m)
    int tm_ok;        // host side: the TMEM Thomas sweep's division ranges hold (k_validate_tm)
    int plane_begin = 0;  // fused stencil sweep only: planes [plane_begin, plane_begin + plane_count)
    int plane_count = 0;  // (0: all m_loc planes); see spmv_plane_ranges
    HaloLink<T> halo;     // fused peer-memory halo (fused_halo_ok); off by default
};

// Reasons a solve stops with NumericalBreakdown (operator.hpp:21-24,
// solver.hpp:214-362).
enum ErrCode { kErrNone = 0,
               kErrPivotFused = 1,    // interleaved_prec_kernel zero pivot
               kErrPivotPrecond = 2,  // precondition zero pivot
               kErrKappa = 3,         // <r,z> not positive
               kErrSigma = 4,         // <p,Ap> not positive
               kErrPivotTridiag = 5 };// solve_tridiag_set zero pivot (CSR backend)

// Device-resident CG scalars and loop control (FusedState<T> scalars,
// operator.hpp:195-208, plus the driver state of solver.hpp:275-370).
template <typename T>
struct Scalars {
    T alpha, beta, kappa, kappa_old, sigma, r_norm, r0, neg_alpha;
    T val[4];  // last reduction results (API queries)
    double eps, tau;
    int maxiter, it, iterations;
    int done, converged, error;
    int n_res, n_kap, n_alp, n_bet;
    int pivot;  // written by the Thomas kernels on a zero pivot (2: stored tridiagonals)
    int hmask;  // history arrays are rings of hmask + 1 entries (the host drains them)
    int pend;   // consumed-reduction mode: the last sweep's tree leaves await their finish
    double* h_res;
    double* h_kap;
    double* h_alp;
    double* h_bet;
};

// Scalar programs run by the reduction finish (all on device, no host sync).
enum ScalarOp {
    kOpStore = 0,     // val[] = sums
    kOpR0 = 1,        // r0 = sqrt(s0); history; tau test     (solver.hpp:299-312)
    kOpKappa0 = 2,    // kappa_old = s0 > 0                     (:317-323)
    kOpSigma0 = 3,    // sigma = s0 > 0; alpha                  (:329-336)
    kOpIlPrec = 4,    // after fused prec: ||r||, kappa, test, beta   (:340-356)
    kOpIlSpmv = 5,    // after fused spmv: sigma, alpha, it++         (:358-364)
    kOpStdSigma = 6,  // standard loop: sigma, alpha                  (:224-230)
    kOpStdRnorm = 7,  // standard loop: ||r||, test                   (:236-244)
    kOpStdKappa = 8,  // standard loop: kappa, beta, it++             (:250-258)
};

// Consumed-reduction mode: instead of a reduction kernel after each sweep,
// every CTA of the NEXT sweep reduces the previous sweep's tree leaves in its
// prologue (the same perfect tree, so the same bits) and runs the scalar
// program on its own copy of the state; CTA (0, 0) writes the result as the
// other state buffer (K1 reads A and writes B, K2 reads B and writes A, so no
// kernel reads what it writes). The last sweep's pending finish runs as one
// tree kernel at the end of a batch of iterations.
template <typename T>
struct Consume {
    const T* leaves;  // the previous sweep's tree leaves (nv arrays of nleaves)
    int nleaves;      // power of two, <= kConsumeMaxLeaves
    int nv;           // 1 or 2
    int op;           // kOpIlSpmv (in K1) or kOpIlPrec (in K2)
    const Scalars<T>* in;
    Scalars<T>* out;
};
constexpr int kConsumeMaxLeaves = 1024;
constexpr long long kConsumeK2Stage = 2LL * 131072;  // K2's leaves: third array of slab.stage

// Fixed-shape pairwise reduction plan (parallel.hpp:11-20) for n values:
// nodes at depth D are summed per thread by the reference's own rule
// (sizes <= 16), everything above depth D is a perfect binary tree.
struct TreePlan {
    long long n;
    int depth;    // D
    int nodes;    // 2^D
    int threads;  // stage-1 block size (<= 256, power of two)
    int blocks;   // stage-1 blocks = stage-2 leaves (power of two)
};
TreePlan make_tree_plan(long long n);

// Dynamic shared memory of one Thomas block (K1/K4) for a column height.
size_t thomas_smem_per_block(int dsize, int n_z, bool global_phi);

// ----------------------------------------------------------------- launchers
extern std::atomic<long long> g_launches;  // kernel launches issued (all entry points)

// The fused sweeps return the number of reduction-tree leaves they wrote to
// `stage` (cta_subtree_sums; stage == nullptr or 0: per-column partials were
// written to part_* and the reduction runs k_tree1).
template <typename T>
int launch_fused_prec(const SlabView<T>& v, bool fast, T* r, T* z, const T* q, T* part_r2,
                      T* part_k, Scalars<T>* S, T* phi_scratch, T* stage, cudaStream_t st,
                      const Consume<T>* cs = nullptr);
// Once per slab: may the sweeps use the TMEM kernel with common-path
// divisions (k_validate_tm)? Synchronous.
template <typename T>
bool validate_thomas_tm(const SlabView<T>& v, cudaStream_t st);
template <typename T>
void launch_precondition(const SlabView<T>& v, bool fast, const T* y, T* x, Scalars<T>* S,
                         const Scalars<T>* gate, T* phi_scratch, cudaStream_t st);
// Can launch_fused_spmv sweep a sub-range of the slab's planes (halo overlap:
// interior planes while the ghost planes are in flight, then the boundary)?
// Most reduction-tree leaves a sweep's fused stage 1 may emit; slab.stage holds
// 3 * max(k_tree1 blocks, kMaxFusedLeaves) values (stage 1.5 writes its nodes
// after the leaves).
constexpr int kMaxFusedLeaves = 131072;
static_assert(kConsumeK2Stage == 2LL * kMaxFusedLeaves, "K2 leaves live in stage's third array");
// Entries per device history ring (Scalars::hmask + 1); the solver loop drains
// them to host vectors, so histories of any length fit (maxiter = 1e9 works).
constexpr int kHistRing = 4096;

// true when the interleaved sweeps chosen for this view honour SlabView::halo
// (K1 = k_thomas_tm default configuration, K2 = k_fused_spmv_pair2).
template <typename T>
bool fused_halo_ok(const SlabView<T>& v, bool fast, bool phi_in_hbm);
template <typename T>
bool spmv_plane_ranges(const SlabView<T>& v, bool fast);
template <typename T>
int launch_fused_spmv(const SlabView<T>& v, bool fast, T* u, T* p, T* q, const T* z, T* part,
                      const Scalars<T>* S, T* stage, cudaStream_t st,
                      const Consume<T>* cs = nullptr);
// Consumed-reduction mode (small single-slab grids): applies when
// both interleaved sweeps are the fused-reduction kernels (fp64 k_thomas_tm,
// k_fused_spmv_pair2) and each emits at most kConsumeMaxLeaves tree leaves;
// returns the two leaf counts.
template <typename T>
bool consume_plan(const SlabView<T>& v, bool phi_in_hbm, int* leaves_k1, int* leaves_k2);
template <typename T>
void launch_apply(const SlabView<T>& v, bool fast, const T* x, T* y, const Scalars<T>* gate,
                  cudaStream_t st);
template <typename T>
void launch_residual_partials(const SlabView<T>& v, bool fast, const T* u, const T* f, T* part,
                              cudaStream_t st);
template <typename T>
void launch_dot_partials(const SlabView<T>& v, const T* x, const T* y, T* part,
                         const Scalars<T>* gate, cudaStream_t st);
// y = c*x + y with c = value (coef == nullptr) or *coef (negated if neg).
template <typename T>
void launch_axpy(long long n, T value, const T* coef, bool neg, const T* x, T* y,
                 const Scalars<T>* gate, cudaStream_t st);
template <typename T>
void launch_scal(long long n, T value, const T* coef, T* x, const Scalars<T>* gate,
                 cudaStream_t st);
template <typename T>
void launch_copy(long long n, const T* x, T* y, const Scalars<T>* gate, cudaStream_t st);
template <typename T>
void launch_fill(long long n, T value, T* x, cudaStream_t st);
template <typename T>
void launch_fill_random(const SlabView<T>& v, uint64_t seed, T* x, cudaStream_t st);

// Matrix-explicit backend (acg_csr.cuh): device assembly of the CSR matrix
// (rows in device order, entries in the caller layout's order) and of the
// stored tridiagonals; spmv_csr; solve_tridiag_set.
template <typename T>
void launch_csr_assemble(const SlabView<T>& v, int horizontal, long long* row_ptr, int* col_idx,
                         T* vals, T* dl, T* dd, T* du, cudaStream_t st);
template <typename T>
void launch_csr_spmv(const SlabView<T>& v, const long long* row_ptr, const int* col_idx,
                     const T* vals, const T* x, T* y, const Scalars<T>* gate, cudaStream_t st);
template <typename T>
void launch_csr_tridiag(const SlabView<T>& v, const T* dl, const T* dd, const T* du, const T* y,
                        T* x, T* phi, Scalars<T>* flag, const Scalars<T>* gate, cudaStream_t st);

// Reductions: nv (<= 3) arrays of plan.n values -> slab sums.
//  stage 1: blocks x nv partial node sums into `stage`.
//  stage 2: perfect tree over the blocks; writes nv slab sums into
//           gather[slab * 4 + v]; if finish, also combines the gather and runs `op`.
template <typename T>
void launch_tree_stage1(const TreePlan& plan, const T* in0, const T* in1, const T* in2, int nv,
                        T* stage, const Scalars<T>* gate, cudaStream_t st);
// Peer-memory ranks: stage 2 also copies the rank's 4 slab sums into every
// rank's mailbox (dst[q] + rank*4) and releases flag[q][rank] = seq. With
// `wait` set, the same kernel then acquires wait[q] >= seq for every rank q,
// combines all ranks' sums from its own mailbox (`all`) and runs the scalar
// program — the whole cross-rank reduction in one launch.
template <typename T>
struct IpcPut {
    T* const* dst;
    unsigned long long* const* flag;
    int n, rank;
    unsigned long long seq;
    const unsigned long long* wait = nullptr;
    const T* all = nullptr;
};
// Returns true when the kernel also finished the reduction (IpcPut::wait).
template <typename T>
bool launch_tree_stage2(const TreePlan& plan, const T* stage, int nv, T* gather, int slab,
                        bool finish, int nslabs, bool exact_tree, Scalars<T>* S, int op,
                        cudaStream_t st, const IpcPut<T>* put = nullptr);
// wait_flags (peer-memory ranks): first wait until wait_flags[q] >= seq for all q < nslabs
template <typename T>
void launch_finish(const T* gather, int nv, int nslabs, bool exact_tree, Scalars<T>* S, int op,
                   cudaStream_t st, const unsigned long long* wait_flags = nullptr,
                   unsigned long long seq = 0);

// Peer-memory (CUDA IPC) transport between the ranks of one node. Flags are
// 64-bit sequence numbers in the owner's mailbox, written by peers with
// system-scope release stores after their data landed, polled with acquire
// loads (a poll that does not complete within ~20 s traps instead of hanging).
//  signal: flags[i] = seq for the non-null entries of flags[0..n)
//  wait:   until flags[i] >= seq for the entries of `need` (bit i)
void launch_ipc_signal(unsigned long long* const* flags, int n, unsigned long long seq,
                       cudaStream_t st);
void launch_ipc_wait(const unsigned long long* flags, int n, unsigned long long need,
                     unsigned long long seq, cudaStream_t st);

// Device-to-host snapshot of `words` 8-byte words into mapped pinned memory by
// a one-warp kernel: stream-ordered like a cudaMemcpyAsync, but it does not
// queue behind bulk DMA on the copy engines (the solve loop's done-flag polls
// while asynchronous field transfers run).
void launch_snapshot(const void* src, void* dst_mapped, int words, cudaStream_t st);

// relayout between the reference's host layouts and plane-major (K7):
// out[x*osx + y + b*osb] = in[x + y*isy + b*isb]  for x<nx, y<ny, b<nb
template <typename T>
void launch_transpose(const T* in, T* out, int nx, int ny, int nb, long long isy, long long isb,
                      long long osx, long long osb, cudaStream_t st);

}  // namespace acg
