// Host runtime of libacg_cuda.so: the C ABI of include/acg.h.
//
// Owns device contexts (profile + per-column geometry per i-slab), fields,
// halo exchange between slabs (device copies on one GPU, NCCL send/recv
// across processes), the exact pairwise reductions, and the device-resident
// PCG drivers (solver.hpp:162-370) whose scalar recurrences run on the GPU so
// the loop never waits on the host.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <unistd.h>
#include <nccl.h>  // types only; NCCL itself is dlopen'ed on first use
#include <nvtx3/nvToolsExt.h>  // header-only; ranges are no-ops without a profiler

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/acg.h"
#include "acg_internal.h"

using namespace acg;

// =================================================================== errors
namespace {

thread_local std::string t_err;

struct Fail {
    acg_status st;
};

[[noreturn]] void fail(acg_status st, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    t_err = buf;
    throw Fail{st};
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(ACG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
#define CK(call) cuda_check((call), #call)

template <typename F>
acg_status guarded(F&& f) {
    try {
        f();
        return ACG_OK;
    } catch (const Fail& e) {
        return e.st;
    } catch (const std::bad_alloc&) {
        t_err = "out of host memory";
        return ACG_ERR_INTERNAL;
    } catch (const std::exception& e) {
        t_err = e.what();
        return ACG_ERR_INTERNAL;
    }
}

// ===================================================================== NCCL
struct NcclApi {
    void* h = nullptr;
    decltype(&::ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&::ncclCommInitRank) commInitRank = nullptr;
    decltype(&::ncclCommDestroy) commDestroy = nullptr;
    decltype(&::ncclCommAbort) commAbort = nullptr;
    decltype(&::ncclGetErrorString) errorString = nullptr;
    decltype(&::ncclAllGather) allGather = nullptr;
    decltype(&::ncclSend) send = nullptr;
    decltype(&::ncclRecv) recv = nullptr;
    decltype(&::ncclGroupStart) groupStart = nullptr;
    decltype(&::ncclGroupEnd) groupEnd = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) return;
#define ACG_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.h, name))
        ACG_SYM(getUniqueId, "ncclGetUniqueId");
        ACG_SYM(commInitRank, "ncclCommInitRank");
        ACG_SYM(commDestroy, "ncclCommDestroy");
        ACG_SYM(commAbort, "ncclCommAbort");
        ACG_SYM(errorString, "ncclGetErrorString");
        ACG_SYM(allGather, "ncclAllGather");
        ACG_SYM(send, "ncclSend");
        ACG_SYM(recv, "ncclRecv");
        ACG_SYM(groupStart, "ncclGroupStart");
        ACG_SYM(groupEnd, "ncclGroupEnd");
#undef ACG_SYM
    });
    if (!api.h || !api.getUniqueId || !api.commInitRank || !api.allGather || !api.send)
        fail(ACG_ERR_NCCL, "NCCL runtime (libnccl.so.2) could not be loaded");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(ACG_ERR_NCCL, "%s: %s", what, nccl().errorString ? nccl().errorString(r) : "error");
}

}  // namespace

struct acg_comm {
    ncclComm_t comm = nullptr;  // NULL after a failed call aborted it (ncclCommAbort)
    int rank = 0, nranks = 1, device = 0;
    int kind = 0;           // 0: NCCL, 1: peer memory (CUDA IPC, one node)
    unsigned char uid[16];  // IPC: rendezvous namespace
    int contexts = 0;       // IPC: contexts created on this communicator (rendezvous key)
};

namespace {

// A failed NCCL call on a communicator aborts it (ncclCommAbort releases the
// other ranks' pending operations instead of leaving them to hang) before the
// error is reported; later calls on the aborted communicator fail immediately.
void nccl_comm_check(acg_comm* c, ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    NcclApi& api = nccl();
    if (c && c->comm && api.commAbort) {
        api.commAbort(c->comm);
        c->comm = nullptr;
    }
    fail(ACG_ERR_NCCL, "%s: %s (communicator aborted)", what,
         api.errorString ? api.errorString(r) : "error");
}

void nccl_comm_alive(const acg_comm* c) {
    if (!c->comm) fail(ACG_ERR_NCCL, "NCCL communicator was aborted after an earlier failure");
}

// Peer-memory transport state of one context (acg_comm_create_ipc). Every rank
// owns a mailbox: flags (halo from below / above, one reduction flag per rank),
// two parities of the two ghost planes, two parities of all ranks' slab sums.
// Peers write into it through CUDA IPC mappings (NVLink P2P between GPUs).
struct IpcState {
    int rank = 0, p = 1;
    char* mbox = nullptr;
    size_t bytes = 0, plane_bytes = 0, off_ghost = 0, off_gather = 0;
    std::vector<char*> peer;  // mailbox of every rank (own = mbox)
    void* dptr = nullptr;     // device: T* sums_dst[2][p], u64* red_flag[p]
    unsigned* arrive = nullptr;  // device [2]: fused-halo CTA arrival counters (HaloLink)
    unsigned long long halo_seq = 0, red_seq = 0;
    std::string file;
    unsigned long long* flags(int q) const { return reinterpret_cast<unsigned long long*>(peer[q]); }
    char* ghost(int q, int parity, int side) const {  // side 0: from below (-1), 1: from above
        return peer[q] + off_ghost + (static_cast<size_t>(parity) * 2 + side) * plane_bytes;
    }
    char* gather(int q, int parity, size_t s) const {
        return peer[q] + off_gather + static_cast<size_t>(parity) * p * 4 * s;
    }
};

std::string hex16(const unsigned char* b) {
    static const char* d = "0123456789abcdef";
    std::string o;
    for (int i = 0; i < 16; ++i) {
        o += d[b[i] >> 4];
        o += d[b[i] & 15];
    }
    return o;
}

struct IpcRecord {
    unsigned magic;
    int rank;
    unsigned long long bytes;
    cudaIpcMemHandle_t handle;
};

// Allocate this rank's mailbox, publish its IPC handle under /dev/shm and map
// every peer's (files keyed by the communicator's id and context ordinal).
std::unique_ptr<IpcState> ipc_attach(acg_comm* comm, long long plane, size_t s) {
    auto st = std::make_unique<IpcState>();
    st->rank = comm->rank;
    st->p = comm->nranks;
    const int p = st->p;
    auto up = [](size_t x) { return (x + 255) / 256 * 256; };
    st->plane_bytes = up(static_cast<size_t>(plane) * s);
    st->off_ghost = up(8 * static_cast<size_t>(2 + p));
    st->off_gather = st->off_ghost + 4 * st->plane_bytes;
    st->bytes = st->off_gather + up(2 * static_cast<size_t>(p) * 4 * s);
    CK(cudaMalloc(&st->mbox, st->bytes));
    CK(cudaMemset(st->mbox, 0, st->bytes));
    CK(cudaDeviceSynchronize());
    IpcRecord rec{0xAC61BC01u, st->rank, st->bytes, {}};
    CK(cudaIpcGetMemHandle(&rec.handle, st->mbox));
    const std::string stem = "/dev/shm/acg-" + hex16(comm->uid) + "-" +
                             std::to_string(comm->contexts++) + "-";
    st->file = stem + std::to_string(st->rank);
    {
        const std::string tmp = st->file + ".tmp";
        FILE* fh = std::fopen(tmp.c_str(), "wb");
        if (!fh || std::fwrite(&rec, sizeof rec, 1, fh) != 1)
            fail(ACG_ERR_INTERNAL, "IPC rendezvous: cannot write %s", tmp.c_str());
        std::fclose(fh);
        if (std::rename(tmp.c_str(), st->file.c_str()) != 0)
            fail(ACG_ERR_INTERNAL, "IPC rendezvous: cannot publish %s", st->file.c_str());
    }
    st->peer.assign(p, nullptr);
    st->peer[st->rank] = st->mbox;
    const auto t0 = std::chrono::steady_clock::now();
    for (int q = 0; q < p; ++q) {
        if (q == st->rank) continue;
        const std::string f = stem + std::to_string(q);
        IpcRecord r{};
        for (;;) {
            FILE* fh = std::fopen(f.c_str(), "rb");
            if (fh) {
                const bool ok = std::fread(&r, sizeof r, 1, fh) == 1;
                std::fclose(fh);
                if (ok && r.magic == rec.magic && r.rank == q) break;
            }
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
                fail(ACG_ERR_INTERNAL, "IPC rendezvous: rank %d never published %s", q, f.c_str());
            std::this_thread::sleep_for(std::chrono::milliseconds(1));
        }
        if (r.bytes != st->bytes)
            fail(ACG_ERR_INVALID_ARGUMENT, "IPC rendezvous: rank %d has a different context", q);
        void* ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, r.handle, cudaIpcMemLazyEnablePeerAccess));
        st->peer[q] = static_cast<char*>(ptr);
    }
    // device pointer tables for the stage-2 put (IpcPut: sums destinations, flags)
    std::vector<void*> tab(3 * static_cast<size_t>(p));
    for (int par = 0; par < 2; ++par)
        for (int q = 0; q < p; ++q) tab[par * p + q] = st->gather(q, par, s);
    for (int q = 0; q < p; ++q) tab[2 * p + q] = st->flags(q) + 2;
    CK(cudaMalloc(&st->arrive, 2 * sizeof(unsigned)));
    CK(cudaMemset(st->arrive, 0, 2 * sizeof(unsigned)));
    CK(cudaMalloc(&st->dptr, tab.size() * sizeof(void*)));
    CK(cudaMemcpy(st->dptr, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice));
    return st;
}

void ipc_detach(IpcState* st) {
    if (!st) return;
    for (int q = 0; q < st->p; ++q)
        if (q != st->rank && st->peer[q]) cudaIpcCloseMemHandle(st->peer[q]);
    if (st->dptr) cudaFree(st->dptr);
    if (st->arrive) cudaFree(st->arrive);
    if (st->mbox) cudaFree(st->mbox);
    if (!st->file.empty()) unlink(st->file.c_str());
}

}  // namespace

// ================================================================== context
namespace {

struct Slab {
    int index = 0;  // global slab index
    int i0 = 0, i1 = 0, m_loc = 0;
    long long plane = 0, n_loc = 0;
    void* prof = nullptr;
    void* col = nullptr;
    void* part[3] = {nullptr, nullptr, nullptr};
    void* stage = nullptr;
    void* phi = nullptr;
    void* staging = nullptr;
    void* tmp = nullptr;  // Scalars<T> for API calls
    TreePlan plan{};
    bool tm_ok = false;   // TMEM Thomas sweep usable (validate_thomas_tm)
    // matrix-explicit backend (acg_csr.cuh), assembled on first use per layout
    int csr_layout = -1;
    long long* csr_rp = nullptr;
    int* csr_ci = nullptr;
    void* csr_val = nullptr;
    void* tri[3] = {nullptr, nullptr, nullptr};  // dl, dd, du (plane-major)
    void* tri_phi = nullptr;
};

void free_csr(Slab& s) {
    void* ps[] = {s.csr_rp, s.csr_ci, s.csr_val, s.tri[0], s.tri[1], s.tri[2], s.tri_phi};
    for (void* p : ps)
        if (p) cudaFree(p);
    s.csr_rp = nullptr;
    s.csr_ci = nullptr;
    s.csr_val = nullptr;
    s.tri[0] = s.tri[1] = s.tri[2] = nullptr;
    s.tri_phi = nullptr;
    s.csr_layout = -1;
}

size_t dsize(acg_dtype t) { return t == ACG_F32 ? sizeof(float) : sizeof(double); }

bool is_pow2(long long x) { return x > 0 && (x & (x - 1)) == 0; }

// Node [lo, hi) of the reference's pairwise tree (parallel.hpp:11-20) at `depth`.
void tree_node(long long n, int depth, long long t, long long& lo, long long& hi) {
    lo = 0;
    hi = n;
    for (int b = depth - 1; b >= 0; --b) {
        const long long mid = lo + (hi - lo) / 2;
        if ((t >> b) & 1)
            lo = mid;
        else
            hi = mid;
    }
}

}  // namespace

struct acg_context {
    acg_dtype dtype = ACG_F64;
    acg_math math = ACG_MATH_EXACT;
    int m = 0, n_z = 0, device = 0;
    int nslabs_total = 1, rank = 0;
    acg_comm* comm = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t halo_stream = nullptr;       // ranks > 1: halo exchange beside the interior sweep
    // asynchronous host transfers (acg_field_upload_async / _download_async):
    // DMA and relayout on their own stream, beside the solver's kernels
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_copy = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
    bool exact_tree = true;
    std::vector<Slab> slabs;  // local slabs (same device)
    void* gather = nullptr;       // nslabs_total * 4 T
    void* gather_send = nullptr;  // 4 T (NCCL)
    std::vector<acg_field*> pool; // reusable scratch fields (host entry points)
    acg_solver* cached = nullptr; // solver state reused by acg_solve / acg_solve_host
    // Serialises every entry point that touches the mutable per-context state
    // above (scratch pool, cached solver, staging buffers, API scalars, the
    // stream's reduction buffers). The reference shares OperatorContext
    // read-only between concurrent solves (operator.hpp:28); here
    // concurrent calls on one context queue on this lock and run one after
    // the other on the context's stream, so each sees a consistent state.
    mutable std::recursive_mutex mu;
    // Fields and solvers the caller created on this context. Destroying the
    // context releases their device memory and orphans them (ctx = NULL), so a
    // later acg_field_destroy / acg_solver_destroy — e.g. from a garbage
    // collector that finalises the context first — frees only the handle.
    mutable std::vector<acg_field*> user_fields;
    mutable std::vector<acg_solver*> user_solvers;
    // pinned double buffer for transfers from / to pageable host memory (lazy)
    mutable void* pin[2] = {nullptr, nullptr};
    mutable cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    std::unique_ptr<IpcState> ipc; // peer-memory transport (acg_comm_create_ipc)
    size_t s = 8;
    bool fast() const { return math == ACG_MATH_FAST; }
};

struct acg_field {
    const acg_context* ctx = nullptr;
    std::vector<void*> base;  // per local slab: (m_loc + 2) planes
    // asynchronous transfers: per-slab staging (allocated on first use) and the
    // event the copy stream records after the field's last async transfer;
    // every entry point that touches the field orders its stream after it
    mutable std::vector<void*> stage;
    mutable cudaEvent_t ev = nullptr;
    mutable bool pending = false;
    void* data(size_t i) const {
        return static_cast<char*>(base[i]) + ctx->slabs[i].plane * ctx->s;
    }
};

namespace {

// NVTX range for profilers (nsys/ncu timelines): init sweeps, iteration
// batches, finish, CSR assembly.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

struct CtxLock {
    std::unique_lock<std::recursive_mutex> lk;
    explicit CtxLock(const acg_context* c) : lk(c->mu) {}
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

template <typename T>
SlabView<T> view(const acg_context* c, size_t si) {
    const Slab& s = c->slabs[si];
    SlabView<T> v;
    v.m = c->m;
    v.n_z = c->n_z;
    v.m_loc = s.m_loc;
    v.i0 = s.i0;
    v.plane = s.plane;
    v.prof = static_cast<const T*>(s.prof);
    v.col = static_cast<const T*>(s.col);
    v.tm_ok = s.tm_ok ? 1 : 0;
    return v;
}

void check_ctx(const acg_context* c) {
    if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "null context");
}
// Work enqueued on `c`'s stream after this call sees the field's asynchronous
// transfers complete (a device-side wait; the host does not block).
void await_field(const acg_context* c, const acg_field* f) {
    if (f && f->pending) CK(cudaStreamWaitEvent(c->stream, f->ev, 0));
}

void check_field(const acg_context* c, const acg_field* f, const char* what) {
    if (!f) fail(ACG_ERR_INVALID_ARGUMENT, "%s: null field", what);
    if (f->ctx != c && !(f->ctx && c && f->ctx->m == c->m && f->ctx->n_z == c->n_z &&
                         f->ctx->slabs.size() == c->slabs.size() && f->ctx->dtype == c->dtype))
        fail(ACG_ERR_INVALID_ARGUMENT, "%s: field does not match operator context", what);
    await_field(c, f);
}

template <typename T>
void build_slab_tables(const acg_context* c, Slab& s, const acg_operator_desc* d) {
    const int m = c->m, n_z = c->n_z;
    std::vector<T> prof(static_cast<size_t>(kProfRows) * n_z);
    for (int k = 0; k < n_z; ++k) {
        // OperatorContext<T> converts each double to T (operator.hpp:36-43); the
        // per-level combination (a'-b')-c' is then formed in T exactly as the
        // kernels of operator.hpp:127/:307 form it.
        const T a = static_cast<T>(d->a_prime[k]), b = static_cast<T>(d->b_prime[k]);
        const T cc = static_cast<T>(d->c_prime[k]), dd = static_cast<T>(d->d[k]);
        volatile T ab = a - b;  // keep the two roundings separate
        prof[kProfS * n_z + k] = static_cast<T>(ab) - cc;
        prof[kProfB * n_z + k] = b;
        prof[kProfC * n_z + k] = cc;
        prof[kProfD * n_z + k] = dd;
        prof[kProfInvD * n_z + k] = T(1) / dd;
    }
    const long long ncol = static_cast<long long>(s.m_loc) * m;
    std::vector<T> col(static_cast<size_t>(kColRows) * ncol);
    for (int il = 0; il < s.m_loc; ++il) {
        const int i = s.i0 + il;
        for (int j = 0; j < m; ++j) {
            const long long ci = static_cast<long long>(il) * m + j;
            const size_t g = static_cast<size_t>(i) * m + j;
            const T area = static_cast<T>(d->cell_area[g]);
            const T adiag = static_cast<T>(d->alpha_diag[g]);
            col[kColArea * ncol + ci] = area;
            col[kColDiag * ncol + ci] = adiag;
            col[kColAtil * ncol + ci] = adiag / area;
            col[kColE * ncol + ci] =
                i + 1 < m ? static_cast<T>(d->alpha_east[static_cast<size_t>(i) * m + j]) : T(0);
            col[kColW * ncol + ci] =
                i > 0 ? static_cast<T>(d->alpha_east[static_cast<size_t>(i - 1) * m + j]) : T(0);
            col[kColN * ncol + ci] =
                j + 1 < m ? static_cast<T>(d->alpha_north[static_cast<size_t>(i) * (m - 1) + j])
                          : T(0);
            col[kColS * ncol + ci] =
                j > 0 ? static_cast<T>(d->alpha_north[static_cast<size_t>(i) * (m - 1) + j - 1])
                      : T(0);
            col[kColInvA * ncol + ci] = T(1) / area;
        }
    }
    CK(cudaMalloc(&s.prof, prof.size() * sizeof(T)));
    CK(cudaMemcpy(s.prof, prof.data(), prof.size() * sizeof(T), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&s.col, col.size() * sizeof(T)));
    CK(cudaMemcpy(s.col, col.data(), col.size() * sizeof(T), cudaMemcpyHostToDevice));
}

void free_slab(Slab& s) {
    free_csr(s);
    void* ps[] = {s.prof, s.col, s.part[0], s.part[1], s.part[2], s.stage, s.phi, s.staging, s.tmp};
    for (void* p : ps)
        if (p) cudaFree(p);
    s = Slab{};
}

// Partition of the m i-planes into p contiguous slabs. When p is a power of
// two and the depth-log2(p) nodes of the reference's column-order pairwise
// tree fall on plane boundaries, those nodes ARE the slabs: every slab then
// sums a complete subtree and the perfect tree above reproduces the CPU sum
// bit for bit.
void partition(int m, int p, std::vector<std::pair<int, int>>& out, bool& exact) {
    out.clear();
    const long long n = static_cast<long long>(m) * m;
    exact = (p == 1);
    if (p > 1 && is_pow2(p)) {
        int depth = 0;
        while ((1 << depth) < p) ++depth;
        bool ok = (n >> (depth - 1)) > 8;  // every node above the slabs is a split node
        std::vector<std::pair<int, int>> cand;
        for (int r = 0; r < p && ok; ++r) {
            long long lo, hi;
            tree_node(n, depth, r, lo, hi);
            if (lo % m || hi % m || hi <= lo) ok = false;
            cand.emplace_back(static_cast<int>(lo / m), static_cast<int>(hi / m));
        }
        if (ok) {
            out = cand;
            exact = true;
            return;
        }
    }
    for (int r = 0; r < p; ++r)
        out.emplace_back(static_cast<int>(static_cast<long long>(r) * m / p),
                         static_cast<int>(static_cast<long long>(r + 1) * m / p));
}

template <typename T>
void* alloc_tmp_scalars() {
    void* p = nullptr;
    CK(cudaMalloc(&p, sizeof(Scalars<T>)));
    CK(cudaMemset(p, 0, sizeof(Scalars<T>)));
    return p;
}

}  // namespace

void destroy_cached_solver(acg_context* c);  // defined after acg_solver
void orphan_solver(acg_solver* s);           // frees a user solver's device state, ctx = NULL
namespace {
void free_pinned(const acg_context* c);      // pinned transfer chunks (defined with h2d/d2h)
void release_field_memory(acg_field* f);  // device memory + async staging (after its transfers)
}  // namespace

// =================================================================== basics
extern "C" {

const char* acg_last_error(void) { return t_err.c_str(); }
int acg_abi_version(void) { return ACG_ABI_VERSION; }
long long acg_kernel_launch_count(void) { return g_launches.load(); }

acg_status acg_device_count(int* count) {
    return guarded([&] {
        if (!count) fail(ACG_ERR_INVALID_ARGUMENT, "null output");
        CK(cudaGetDeviceCount(count));
    });
}

acg_status acg_host_alloc(void** ptr, size_t bytes) {
    return guarded([&] {
        if (!ptr) fail(ACG_ERR_INVALID_ARGUMENT, "null output");
        CK(cudaHostAlloc(ptr, bytes ? bytes : 1, cudaHostAllocPortable));
    });
}

acg_status acg_host_free(void* ptr) {
    return guarded([&] {
        if (ptr) CK(cudaFreeHost(ptr));
    });
}

acg_status acg_comm_unique_id(void* id128) {
    return guarded([&] {
        if (!id128) fail(ACG_ERR_INVALID_ARGUMENT, "null output");
        ncclUniqueId id;
        nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id128, &id, sizeof(id));
    });
}

acg_status acg_comm_create(acg_comm** out, int rank, int nranks, const void* id128, int device) {
    return guarded([&] {
        if (!out || !id128) fail(ACG_ERR_INVALID_ARGUMENT, "null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks)
            fail(ACG_ERR_INVALID_ARGUMENT, "bad rank %d of %d", rank, nranks);
        DeviceGuard g(device);
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        auto c = std::make_unique<acg_comm>();
        c->rank = rank;
        c->nranks = nranks;
        c->device = device;
        nccl_check(nccl().commInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
        *out = c.release();
    });
}

acg_status acg_comm_create_ipc(acg_comm** out, int rank, int nranks, const void* id128,
                               int device) {
    return guarded([&] {
        if (!out || !id128) fail(ACG_ERR_INVALID_ARGUMENT, "null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks)
            fail(ACG_ERR_INVALID_ARGUMENT, "bad rank %d of %d", rank, nranks);
        auto c = std::make_unique<acg_comm>();
        c->rank = rank;
        c->nranks = nranks;
        c->device = device;
        c->kind = 1;
        std::memcpy(c->uid, id128, sizeof c->uid);
        *out = c.release();
    });
}

acg_status acg_comm_destroy(acg_comm* c) {
    return guarded([&] {
        if (!c) return;
        if (c->comm) nccl().commDestroy(c->comm);
        delete c;
    });
}

acg_status acg_context_create(acg_context** out, acg_dtype dtype, const acg_operator_desc* d,
                              const acg_placement* pl) {
    return guarded([&] {
        if (!out || !d) fail(ACG_ERR_INVALID_ARGUMENT, "null argument");
        if (d->m < 1 || d->n_z < 1)
            fail(ACG_ERR_INVALID_ARGUMENT, "OperatorContext: empty profile or geometry");
        if (dtype != ACG_F64 && dtype != ACG_F32) fail(ACG_ERR_INVALID_ARGUMENT, "bad dtype");
        if (!d->a_prime || !d->b_prime || !d->c_prime || !d->d || !d->cell_area || !d->alpha_diag ||
            (d->m > 1 && (!d->alpha_east || !d->alpha_north)))
            fail(ACG_ERR_INVALID_ARGUMENT, "OperatorContext: missing coefficient array");
        auto c = std::make_unique<acg_context>();
        c->dtype = dtype;
        c->s = dsize(dtype);
        c->m = d->m;
        c->n_z = d->n_z;
        int p = 1;
        if (pl) {
            c->math = pl->math;
            c->device = pl->device;
            c->comm = pl->comm;
            if (pl->comm) {
                p = pl->comm->nranks;
                c->rank = pl->comm->rank;
                if (pl->comm->device != pl->device)
                    fail(ACG_ERR_INVALID_ARGUMENT, "placement device differs from comm device");
            } else {
                p = pl->slabs < 1 ? 1 : pl->slabs;
            }
        } else {
            cudaGetDevice(&c->device);
        }
        if (p > d->m) fail(ACG_ERR_INVALID_ARGUMENT, "more slabs (%d) than i-planes (%d)", p, d->m);
        if (p > 64) fail(ACG_ERR_INVALID_ARGUMENT, "at most 64 slabs are supported");
        c->nslabs_total = p;
        DeviceGuard g(c->device);
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        std::vector<std::pair<int, int>> parts;
        partition(d->m, p, parts, c->exact_tree);
        std::vector<int> mine;
        if (c->comm)
            mine.push_back(c->rank);
        else
            for (int r = 0; r < p; ++r) mine.push_back(r);
        c->slabs.resize(mine.size());
        for (size_t a = 0; a < mine.size(); ++a) {
            Slab& s = c->slabs[a];
            s.index = mine[a];
            s.i0 = parts[mine[a]].first;
            s.i1 = parts[mine[a]].second;
            s.m_loc = s.i1 - s.i0;
            s.plane = static_cast<long long>(d->n_z) * d->m;
            s.n_loc = s.plane * s.m_loc;
            if (dtype == ACG_F32) {
                build_slab_tables<float>(c.get(), s, d);
                s.tmp = alloc_tmp_scalars<float>();
                s.tm_ok = validate_thomas_tm<float>(view<float>(c.get(), a), c->stream);
            } else {
                build_slab_tables<double>(c.get(), s, d);
                s.tmp = alloc_tmp_scalars<double>();
                s.tm_ok = validate_thomas_tm<double>(view<double>(c.get(), a), c->stream);
            }
            const long long ncol = static_cast<long long>(s.m_loc) * d->m;
            for (int a2 = 0; a2 < 3; ++a2) CK(cudaMalloc(&s.part[a2], ncol * c->s));
            s.plan = make_tree_plan(ncol);
            if (s.plan.blocks > 16384)
                fail(ACG_ERR_INVALID_ARGUMENT, "slab of %lld columns exceeds the reduction plan",
                     ncol);
            // stage: k_tree1 block sums, or up to kMaxFusedLeaves node sums written by a
            // sweep followed by the stage-1.5 nodes
            CK(cudaMalloc(&s.stage,
                          3 * static_cast<size_t>(std::max(s.plan.blocks, kMaxFusedLeaves)) * c->s));
            if (thomas_smem_per_block(static_cast<int>(c->s), d->n_z, false) > 200 * 1024)
                CK(cudaMalloc(&s.phi, s.n_loc * c->s));  // tall columns: phi in HBM
        }
        CK(cudaMalloc(&c->gather, static_cast<size_t>(p) * 4 * c->s));
        CK(cudaMemset(c->gather, 0, static_cast<size_t>(p) * 4 * c->s));
        CK(cudaMalloc(&c->gather_send, 4 * c->s));
        if (c->comm && c->comm->kind == 1 && p > 1)
            c->ipc = ipc_attach(c->comm, c->slabs[0].plane, c->s);
        if (c->comm && p > 1) {
            CK(cudaStreamCreateWithFlags(&c->halo_stream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
        }
        *out = c.release();
    });
}

acg_status acg_partition_plan(int m, int p, int* i_begin, int* exact_tree) {
    return guarded([&] {
        if (m < 1 || p < 1 || p > m || !i_begin || !exact_tree)
            fail(ACG_ERR_INVALID_ARGUMENT, "partition_plan: bad arguments");
        std::vector<std::pair<int, int>> parts;
        bool exact = false;
        partition(m, p, parts, exact);
        for (int s = 0; s < p; ++s) i_begin[s] = parts[s].first;
        i_begin[p] = parts[p - 1].second;
        *exact_tree = exact ? 1 : 0;
    });
}

acg_status acg_context_destroy(acg_context* c) {
    return guarded([&] {
        if (!c) return;
        DeviceGuard g(c->device);
        cudaStreamSynchronize(c->stream);
        for (acg_solver* us : c->user_solvers) orphan_solver(us);
        for (acg_field* f : c->user_fields) {
            release_field_memory(f);
            if (f->ev) cudaEventDestroy(f->ev);
            f->ev = nullptr;
            f->ctx = nullptr;
        }
        destroy_cached_solver(c);
        for (acg_field* f : c->pool) {
            for (void* b : f->base) cudaFree(b);
            delete f;
        }
        for (Slab& s : c->slabs) free_slab(s);
        free_pinned(c);
        if (c->gather) cudaFree(c->gather);
        if (c->gather_send) cudaFree(c->gather_send);
        ipc_detach(c->ipc.get());
        if (c->halo_stream) cudaStreamDestroy(c->halo_stream);
        if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
        if (c->ev_copy) cudaEventDestroy(c->ev_copy);
        if (c->ev_ready) cudaEventDestroy(c->ev_ready);
        if (c->ev_halo) cudaEventDestroy(c->ev_halo);
        if (c->stream) cudaStreamDestroy(c->stream);
        delete c;
    });
}

acg_status acg_context_info_get(const acg_context* c, acg_context_info* o) {
    return guarded([&] {
        check_ctx(c);
        if (!o) fail(ACG_ERR_INVALID_ARGUMENT, "null output");
        o->m = c->m;
        o->n_z = c->n_z;
        o->dtype = c->dtype;
        o->math = c->math;
        o->nslabs_total = c->nslabs_total;
        o->nslabs_local = static_cast<int>(c->slabs.size());
        o->rank = c->rank;
        o->i_begin = c->slabs.front().i0;
        o->i_end = c->slabs.back().i1;
        o->exact_tree = c->exact_tree ? 1 : 0;
        size_t b = 0;
        for (const Slab& s : c->slabs) b += static_cast<size_t>(s.n_loc) * c->s;
        o->bytes_per_field_local = b;
        o->thomas_tmem = 1;
        for (const Slab& s : c->slabs)
            if (!s.tm_ok) o->thomas_tmem = 0;
    });
}

acg_status acg_synchronize(const acg_context* c) {
    return guarded([&] {
        check_ctx(c);
        DeviceGuard g(c->device);
        CtxLock lk(c);
        CK(cudaStreamSynchronize(c->stream));
        if (c->copy_stream) CK(cudaStreamSynchronize(c->copy_stream));
    });
}

void* acg_context_stream(const acg_context* c) { return c ? c->stream : nullptr; }

acg_status acg_context_wait_stream(const acg_context* c, void* stream) {
    return guarded([&] {
        check_ctx(c);
        DeviceGuard g(c->device);
        CtxLock lk(c);
        cudaEvent_t e = nullptr;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        const cudaError_t r1 = cudaEventRecord(e, static_cast<cudaStream_t>(stream));
        const cudaError_t r2 = r1 == cudaSuccess ? cudaStreamWaitEvent(c->stream, e, 0) : r1;
        cudaEventDestroy(e);  // released once the wait is resolved
        CK(r2);
    });
}

acg_status acg_stream_wait_context(void* stream, const acg_context* c) {
    return guarded([&] {
        check_ctx(c);
        DeviceGuard g(c->device);
        CtxLock lk(c);
        cudaEvent_t e = nullptr;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        const cudaError_t r1 = cudaEventRecord(e, c->stream);
        const cudaError_t r2 =
            r1 == cudaSuccess ? cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), e, 0) : r1;
        cudaEventDestroy(e);
        CK(r2);
    });
}

acg_status acg_context_release_scratch(const acg_context* cc) {
    return guarded([&] {
        check_ctx(cc);
        DeviceGuard g(cc->device);
        CtxLock lk(cc);
        acg_context* c = const_cast<acg_context*>(cc);
        CK(cudaStreamSynchronize(c->stream));
        if (c->copy_stream) CK(cudaStreamSynchronize(c->copy_stream));
        for (acg_field* f : c->user_fields) {  // async-transfer staging
            for (void* b : f->stage) cudaFree(b);
            f->stage.clear();
        }
        destroy_cached_solver(c);
        for (acg_field* f : c->pool) {
            for (void* b : f->base) cudaFree(b);
            delete f;
        }
        c->pool.clear();
        for (Slab& s : c->slabs) {
            if (s.staging) {
                cudaFree(s.staging);
                s.staging = nullptr;
            }
            free_csr(s);
        }
        free_pinned(c);
    });
}

}  // extern "C"

// ==================================================================== fields
namespace {

// zero_all: the public Field3D contract (zero-filled); internal work fields only
// need their two ghost planes cleared (the owned planes are always written first).
acg_field* new_field(const acg_context* c, bool zero_all = true) {
    auto f = std::make_unique<acg_field>();
    f->ctx = c;
    for (const Slab& s : c->slabs) {
        void* p = nullptr;
        const size_t bytes = static_cast<size_t>(s.n_loc + 2 * s.plane) * c->s;
        const size_t pb = static_cast<size_t>(s.plane) * c->s;
        CK(cudaMalloc(&p, bytes));
        f->base.push_back(p);
        if (zero_all) {
            CK(cudaMemsetAsync(p, 0, bytes, c->stream));
        } else {
            CK(cudaMemsetAsync(p, 0, pb, c->stream));
            CK(cudaMemsetAsync(static_cast<char*>(p) + bytes - pb, 0, pb, c->stream));
        }
    }
    return f.release();
}

// Device memory of a field (its async transfers complete first).
void release_field_memory(acg_field* f) {
    if (f->ev) cudaEventSynchronize(f->ev);
    for (void* b : f->base) cudaFree(b);
    f->base.clear();
    for (void* b : f->stage) cudaFree(b);
    f->stage.clear();
    f->pending = false;
}

void free_field(acg_field* f) {
    release_field_memory(f);
    if (f->ev) cudaEventDestroy(f->ev);
    delete f;
}

struct PoolField {
    acg_context* c;
    acg_field* f;
    explicit PoolField(const acg_context* cc) : c(const_cast<acg_context*>(cc)) {
        if (!c->pool.empty()) {
            f = c->pool.back();
            c->pool.pop_back();
        } else {
            f = new_field(c);
        }
    }
    ~PoolField() { c->pool.push_back(f); }
};

void* staging(const acg_context* c, size_t si) {
    Slab& s = const_cast<Slab&>(c->slabs[si]);
    if (!s.staging) CK(cudaMalloc(&s.staging, static_cast<size_t>(s.n_loc) * c->s));
    return s.staging;
}

// ------------------------------------------------- host <-> device transfers
// Pinned (page-locked or registered) host buffers go straight to the DMA
// engine. Ordinary pageable buffers (numpy arrays through the Python API)
// move through two pinned chunks: host threads copy chunk c+1 while the DMA
// engine moves chunk c. Measured for 1 GB (scripts/micro/h2d_paths.cu): H2D
// 96 ms pageable -> 34 ms staged; D2H 505-526 ms -> 77-83 ms.
constexpr size_t kPinChunk = size_t(32) << 20;

bool host_is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Host threads for the staged copies: persistent workers (spawning a dozen
// threads per 32 MB chunk cost several ms per GB), one job at a time; the
// caller copies slice 0 itself.
class CopyPool {
public:
    explicit CopyPool(int workers) {
        for (int w = 0; w < workers; ++w) th_.emplace_back([this, w] { run(w + 1); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> l(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void copy(char* dst, const char* src, size_t n) {
        std::lock_guard<std::mutex> one_job(job_mu_);
        const size_t parts = th_.size() + 1;
        const size_t per = (n + parts - 1) / parts;
        {
            std::lock_guard<std::mutex> l(m_);
            dst_ = dst;
            src_ = src;
            n_ = n;
            per_ = per;
            pending_ = static_cast<int>(th_.size());
            ++gen_;
        }
        cv_.notify_all();
        std::memcpy(dst, src, std::min(n, per));
        std::unique_lock<std::mutex> l(m_);
        done_.wait(l, [&] { return pending_ == 0; });
    }

private:
    void run(size_t part) {
        unsigned long long seen = 0;
        for (;;) {
            char* dst;
            const char* src;
            size_t n, per;
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                dst = dst_;
                src = src_;
                n = n_;
                per = per_;
            }
            const size_t a = part * per, b = std::min(n, a + per);
            if (a < b) std::memcpy(dst + a, src + a, b - a);
            std::lock_guard<std::mutex> l(m_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> th_;
    std::mutex job_mu_, m_;
    std::condition_variable cv_, done_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t n_ = 0, per_ = 0;
    int pending_ = 0;
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

void par_memcpy(void* dst, const void* src, size_t n) {
    // up to 12 host threads: on the 16-core gpurun hosts a 1 GB numpy solve's
    // staged transfers took ~305 ms end to end with 8, ~292 with 12, ~302 with 16
    static const int nt = [] {
        const unsigned hw = std::thread::hardware_concurrency();
        return static_cast<int>(hw == 0 ? 1 : (hw > 12 ? 12 : hw));
    }();
    if (nt == 1 || n < (size_t(1) << 20)) {
        std::memcpy(dst, src, n);
        return;
    }
    static CopyPool pool(nt - 1);
    pool.copy(static_cast<char*>(dst), static_cast<const char*>(src), n);
}

void ensure_pinned(const acg_context* c) {
    if (c->pin[0]) return;
    for (int b = 0; b < 2; ++b) {
        CK(cudaHostAlloc(&c->pin[b], kPinChunk, cudaHostAllocPortable));
        CK(cudaEventCreateWithFlags(&c->pin_ev[b], cudaEventDisableTiming));
        CK(cudaEventRecord(c->pin_ev[b], c->stream));
    }
}

void free_pinned(const acg_context* c) {
    for (int b = 0; b < 2; ++b) {
        if (c->pin_ev[b]) cudaEventSynchronize(c->pin_ev[b]);
        if (c->pin[b]) cudaFreeHost(c->pin[b]);
        if (c->pin_ev[b]) cudaEventDestroy(c->pin_ev[b]);
        c->pin[b] = nullptr;
        c->pin_ev[b] = nullptr;
    }
}

// Enqueue host -> device (contiguous) on the context's stream; returns once
// `host` may be reused.
void h2d(const acg_context* c, void* dev, const void* host, size_t n) {
    if (n < 2 * kPinChunk || host_is_pinned(host)) {
        CK(cudaMemcpyAsync(dev, host, n, cudaMemcpyHostToDevice, c->stream));
        return;
    }
    ensure_pinned(c);
    int k = 0;
    for (size_t off = 0; off < n; off += kPinChunk, ++k) {
        const size_t len = std::min(kPinChunk, n - off);
        CK(cudaEventSynchronize(c->pin_ev[k & 1]));  // the DMA that used this chunk is done
        par_memcpy(c->pin[k & 1], static_cast<const char*>(host) + off, len);
        CK(cudaMemcpyAsync(static_cast<char*>(dev) + off, c->pin[k & 1], len,
                           cudaMemcpyHostToDevice, c->stream));
        CK(cudaEventRecord(c->pin_ev[k & 1], c->stream));
    }
}

// Device -> host (contiguous) after the work enqueued so far; complete on return.
void d2h(const acg_context* c, void* host, const void* dev, size_t n) {
    if (n < 2 * kPinChunk || host_is_pinned(host)) {
        CK(cudaMemcpyAsync(host, dev, n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return;
    }
    ensure_pinned(c);
    const size_t nch = (n + kPinChunk - 1) / kPinChunk;
    auto issue = [&](size_t ch) {
        const size_t off = ch * kPinChunk, len = std::min(kPinChunk, n - off);
        CK(cudaMemcpyAsync(c->pin[ch & 1], static_cast<const char*>(dev) + off, len,
                           cudaMemcpyDeviceToHost, c->stream));
        CK(cudaEventRecord(c->pin_ev[ch & 1], c->stream));
    };
    issue(0);
    issue(1);
    for (size_t ch = 0; ch < nch; ++ch) {
        const size_t off = ch * kPinChunk, len = std::min(kPinChunk, n - off);
        CK(cudaEventSynchronize(c->pin_ev[ch & 1]));
        par_memcpy(static_cast<char*>(host) + off, c->pin[ch & 1], len);
        if (ch + 2 < nch) issue(ch + 2);
    }
}

// Asynchronous transfers run on the context's copy stream (created on first
// use) with the field's own staging, so they overlap the solver's kernels.
cudaStream_t copy_stream(const acg_context* cc) {
    acg_context* c = const_cast<acg_context*>(cc);
    if (!c->copy_stream) {
        CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming));
    }
    return c->copy_stream;
}

// The copy stream starts after the work enqueued on the context's stream so
// far (earlier kernels may still read or write the field).
cudaStream_t begin_async(const acg_field* f, const void* host, const char* what) {
    const acg_context* c = f->ctx;
    if (!host_is_pinned(host))
        fail(ACG_ERR_INVALID_ARGUMENT,
             "%s: the host buffer is not page-locked (acg_host_alloc / cudaHostAlloc / "
             "cudaHostRegister); use the synchronous call for pageable memory", what);
    cudaStream_t cs = copy_stream(c);
    CK(cudaEventRecord(c->ev_copy, c->stream));
    CK(cudaStreamWaitEvent(cs, c->ev_copy, 0));
    if (!f->ev) CK(cudaEventCreateWithFlags(&f->ev, cudaEventDisableTiming));
    if (f->stage.empty())
        for (const Slab& sl : c->slabs) {
            void* p = nullptr;
            CK(cudaMalloc(&p, static_cast<size_t>(sl.n_loc) * c->s));
            f->stage.push_back(p);
        }
    return cs;
}

// The copy engines serve the DMA commands of all streams in order: one 1 GB
// command would hold the solver's small scalar reads (the done-flag polls,
// history drains) for ~20 ms, so async transfers go in 8 MB pieces (~0.15 ms
// each at PCIe 5 rates).
void dma_chunked(void* dst, const void* src, size_t n, cudaMemcpyKind kind, cudaStream_t st) {
    constexpr size_t kChunk = size_t(8) << 20;
    for (size_t off = 0; off < n; off += kChunk)
        CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off,
                           std::min(kChunk, n - off), kind, st));
}

void end_async(const acg_field* f, cudaStream_t cs) {
    CK(cudaEventRecord(f->ev, cs));
    f->pending = true;
}

// Host -> field: the DMA into a staging buffer, then the relayout kernel. The
// synchronous path (async = false) uses the context's stream and staging and
// accepts pageable memory (h2d); the asynchronous one the copy stream and the
// field's staging, with page-locked memory only.
template <typename T>
void upload_t(acg_field* f, const void* host, acg_layout layout, acg_host_scope scope,
              bool async = false) {
    const acg_context* c = f->ctx;
    const int m = c->m, n_z = c->n_z;
    cudaStream_t st = async ? begin_async(f, host, "upload_async") : c->stream;
    auto copy = [&](void* dst, const void* src, size_t n) {
        if (async)
            dma_chunked(dst, src, n, cudaMemcpyHostToDevice, st);
        else
            h2d(c, dst, src, n);
    };
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        const Slab& s = c->slabs[si];
        T* stg = static_cast<T*>(async ? f->stage[si] : staging(c, si));
        T* dst = static_cast<T*>(f->data(si));
        if (layout == ACG_LAYOUT_VERTICAL) {
            const T* src = static_cast<const T*>(host) +
                           (scope == ACG_HOST_FULL ? static_cast<size_t>(s.i0) * m * n_z : 0);
            copy(stg, src, static_cast<size_t>(s.n_loc) * sizeof(T));
            // stg[(il*m + j)*n_z + k] -> dst[il*plane + k*m + j]
            launch_transpose<T>(stg, dst, n_z, m, s.m_loc, n_z, static_cast<long long>(m) * n_z, m,
                                s.plane, st);
        } else {
            if (scope == ACG_HOST_FULL && s.m_loc != m) {  // strided rows of this slab
                CK(cudaMemcpy2DAsync(stg, s.m_loc * sizeof(T),
                                     static_cast<const T*>(host) + s.i0, m * sizeof(T),
                                     s.m_loc * sizeof(T), static_cast<size_t>(m) * n_z,
                                     cudaMemcpyHostToDevice, st));
            } else {
                copy(stg, host, static_cast<size_t>(s.n_loc) * sizeof(T));
            }
            // stg[(j*n_z + k)*m_loc + il] -> dst[il*plane + k*m + j]
            launch_transpose<T>(stg, dst, s.m_loc, m, n_z, static_cast<long long>(n_z) * s.m_loc,
                                s.m_loc, s.plane, m, st);
        }
        CK(cudaPeekAtLastError());
    }
    if (async) end_async(f, st);
}

// Field -> host; the synchronous path returns with the host buffer complete,
// the asynchronous one after enqueueing (acg_field_wait completes it).
template <typename T>
void download_t(const acg_field* f, void* host, acg_layout layout, acg_host_scope scope,
                bool async = false) {
    const acg_context* c = f->ctx;
    const int m = c->m, n_z = c->n_z;
    cudaStream_t st = async ? begin_async(f, host, "download_async") : c->stream;
    auto copy = [&](void* dst, const void* src, size_t n) {
        if (async)
            dma_chunked(dst, src, n, cudaMemcpyDeviceToHost, st);
        else
            d2h(c, dst, src, n);
    };
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        const Slab& s = c->slabs[si];
        T* stg = static_cast<T*>(async ? f->stage[si] : staging(c, si));
        const T* src = static_cast<const T*>(f->data(si));
        if (layout == ACG_LAYOUT_VERTICAL) {
            // src[il*plane + k*m + j] -> stg[(il*m + j)*n_z + k]
            launch_transpose<T>(src, stg, m, n_z, s.m_loc, m, s.plane, n_z,
                                static_cast<long long>(m) * n_z, st);
            T* dst = static_cast<T*>(host) +
                     (scope == ACG_HOST_FULL ? static_cast<size_t>(s.i0) * m * n_z : 0);
            copy(dst, stg, static_cast<size_t>(s.n_loc) * sizeof(T));
        } else {
            // src[il*plane + k*m + j] -> stg[(j*n_z + k)*m_loc + il]
            launch_transpose<T>(src, stg, m, s.m_loc, n_z, s.plane, m,
                                static_cast<long long>(n_z) * s.m_loc, s.m_loc, st);
            if (scope == ACG_HOST_FULL && s.m_loc != m) {
                CK(cudaMemcpy2DAsync(static_cast<T*>(host) + s.i0, m * sizeof(T), stg,
                                     s.m_loc * sizeof(T), s.m_loc * sizeof(T),
                                     static_cast<size_t>(m) * n_z, cudaMemcpyDeviceToHost, st));
            } else {
                copy(host, stg, static_cast<size_t>(s.n_loc) * sizeof(T));
            }
        }
    }
    if (async)
        end_async(f, st);
    else
        CK(cudaStreamSynchronize(c->stream));
}

// Device-resident counterparts (the Python edge hands over torch/CuPy device
// buffers): the relayout kernel reads / writes the caller's buffer directly,
// no staging and no PCIe traffic.
template <typename T>
void upload_dev_t(acg_field* f, const void* dev, acg_layout layout, acg_host_scope scope) {
    const acg_context* c = f->ctx;
    const int m = c->m, n_z = c->n_z;
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        const Slab& s = c->slabs[si];
        T* dst = static_cast<T*>(f->data(si));
        const T* src = static_cast<const T*>(dev);
        if (layout == ACG_LAYOUT_VERTICAL) {
            if (scope == ACG_HOST_FULL) src += static_cast<size_t>(s.i0) * m * n_z;
            launch_transpose<T>(src, dst, n_z, m, s.m_loc, n_z, static_cast<long long>(m) * n_z, m,
                                s.plane, c->stream);
        } else if (scope == ACG_HOST_FULL) {  // src[(j*n_z + k)*m + i0 + il]
            launch_transpose<T>(src + s.i0, dst, s.m_loc, m, n_z, static_cast<long long>(n_z) * m,
                                m, s.plane, m, c->stream);
        } else {
            launch_transpose<T>(src, dst, s.m_loc, m, n_z, static_cast<long long>(n_z) * s.m_loc,
                                s.m_loc, s.plane, m, c->stream);
        }
        CK(cudaPeekAtLastError());
    }
}

template <typename T>
void download_dev_t(const acg_field* f, void* dev, acg_layout layout, acg_host_scope scope) {
    const acg_context* c = f->ctx;
    const int m = c->m, n_z = c->n_z;
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        const Slab& s = c->slabs[si];
        const T* src = static_cast<const T*>(f->data(si));
        T* dst = static_cast<T*>(dev);
        if (layout == ACG_LAYOUT_VERTICAL) {
            if (scope == ACG_HOST_FULL) dst += static_cast<size_t>(s.i0) * m * n_z;
            launch_transpose<T>(src, dst, m, n_z, s.m_loc, m, s.plane, n_z,
                                static_cast<long long>(m) * n_z, c->stream);
        } else if (scope == ACG_HOST_FULL) {  // dst[(j*n_z + k)*m + i0 + il]
            launch_transpose<T>(src, dst + s.i0, m, s.m_loc, n_z, s.plane, m,
                                static_cast<long long>(n_z) * m, m, c->stream);
        } else {
            launch_transpose<T>(src, dst, m, s.m_loc, n_z, s.plane, m,
                                static_cast<long long>(n_z) * s.m_loc, s.m_loc, c->stream);
        }
        CK(cudaPeekAtLastError());
    }
}

// ---------------------------------------------------------------- halos
// Ghost plane -1 of slab s <- plane m_loc-1 of slab s-1; ghost plane m_loc of
// slab s <- plane 0 of slab s+1. Device copies between local slabs, NCCL
// send/recv between ranks.
void halo(const acg_context* c, const acg_field* f, cudaStream_t hs = nullptr) {
    if (!hs) hs = c->stream;
    if (c->nslabs_total == 1) return;
    const size_t pb = static_cast<size_t>(c->slabs[0].plane) * c->s;
    auto plane_ptr = [&](size_t si, int il) {
        return static_cast<char*>(f->base[si]) + static_cast<size_t>(il + 1) * pb;
    };
    if (!c->comm) {
        for (size_t si = 1; si < c->slabs.size(); ++si) {
            const Slab& lo = c->slabs[si - 1];
            const Slab& hi = c->slabs[si];
            CK(cudaMemcpyAsync(plane_ptr(si, -1), plane_ptr(si - 1, lo.m_loc - 1), pb,
                               cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaMemcpyAsync(plane_ptr(si - 1, lo.m_loc), plane_ptr(si, 0), pb,
                               cudaMemcpyDeviceToDevice, c->stream));
            (void)hi;
        }
        return;
    }
    if (c->ipc) {  // peer memory: write the boundary planes into the neighbours' mailboxes
        IpcState& ip = *c->ipc;
        const int r = ip.rank, p = ip.p, m_loc = c->slabs[0].m_loc;
        const unsigned long long seq = ++ip.halo_seq;
        const int par = static_cast<int>(seq & 1);
        unsigned long long* fl[2] = {nullptr, nullptr};
        if (r > 0) {  // my plane 0 is the ghost "from above" of rank r-1
            CK(cudaMemcpyAsync(ip.ghost(r - 1, par, 1), plane_ptr(0, 0), pb, cudaMemcpyDeviceToDevice,
                               hs));
            fl[0] = ip.flags(r - 1) + 1;
        }
        if (r + 1 < p) {  // my last plane is the ghost "from below" of rank r+1
            CK(cudaMemcpyAsync(ip.ghost(r + 1, par, 0), plane_ptr(0, m_loc - 1), pb,
                               cudaMemcpyDeviceToDevice, hs));
            fl[1] = ip.flags(r + 1) + 0;
        }
        launch_ipc_signal(fl, 2, seq, hs);
        launch_ipc_wait(ip.flags(r), 2, (r > 0 ? 1ull : 0ull) | (r + 1 < p ? 2ull : 0ull), seq,
                        hs);
        if (r > 0)
            CK(cudaMemcpyAsync(plane_ptr(0, -1), ip.ghost(r, par, 0), pb, cudaMemcpyDeviceToDevice,
                               hs));
        if (r + 1 < p)
            CK(cudaMemcpyAsync(plane_ptr(0, m_loc), ip.ghost(r, par, 1), pb,
                               cudaMemcpyDeviceToDevice, hs));
        return;
    }
    NcclApi& api = nccl();
    const int r = c->rank, p = c->nslabs_total;
    const Slab& s = c->slabs[0];
    const ncclDataType_t dt = c->dtype == ACG_F32 ? ncclFloat32 : ncclFloat64;
    const size_t cnt = static_cast<size_t>(s.plane);
    acg_comm* cm = c->comm;
    nccl_comm_alive(cm);
    nccl_comm_check(cm, api.groupStart(), "ncclGroupStart");
    if (r > 0) {
        nccl_comm_check(cm, api.send(plane_ptr(0, 0), cnt, dt, r - 1, cm->comm, hs), "ncclSend");
        nccl_comm_check(cm, api.recv(plane_ptr(0, -1), cnt, dt, r - 1, cm->comm, hs), "ncclRecv");
    }
    if (r + 1 < p) {
        nccl_comm_check(cm, api.send(plane_ptr(0, s.m_loc - 1), cnt, dt, r + 1, cm->comm, hs),
                        "ncclSend");
        nccl_comm_check(cm, api.recv(plane_ptr(0, s.m_loc), cnt, dt, r + 1, cm->comm, hs),
                        "ncclRecv");
    }
    nccl_comm_check(cm, api.groupEnd(), "ncclGroupEnd");
}

// -------------------------------------------------------------- reductions
// Reduce nv per-column partial arrays of every local slab (already written to
// slab.part[0..nv)) and run scalar program `op` on every slab's Scalars.
// leaves[si] > 0: the sweep already wrote that many aligned tree-node sums to
// slab.stage (fused stage 1), so only the perfect tree above them remains.
template <typename T>
void reduce(const acg_context* c, int nv, int op, const std::vector<Scalars<T>*>& S,
            const Scalars<T>* gate_or_null, bool gated, const std::vector<int>* leaves = nullptr) {
    const bool single = c->nslabs_total == 1;
    T* gather = static_cast<T*>(c->gather);
    // peer memory: stage 2 puts the slab sums into every mailbox, the finish waits for them
    IpcPut<T> put{nullptr, nullptr, 0, 0, 0};
    unsigned long long seq = 0;
    int par = 0;
    if (c->ipc && !single) {
        IpcState& ip = *c->ipc;
        seq = ++ip.red_seq;
        par = static_cast<int>(seq & 1);
        put.dst = static_cast<T* const*>(ip.dptr) + static_cast<size_t>(par) * ip.p;
        put.flag = reinterpret_cast<unsigned long long* const*>(static_cast<void* const*>(ip.dptr) +
                                                                2 * ip.p);
        put.n = ip.p;
        put.rank = ip.rank;
        put.seq = seq;
        if (c->slabs.size() == 1) {  // the stage-2 kernel also waits, combines and finishes
            put.wait = ip.flags(ip.rank) + 2;
            put.all = reinterpret_cast<const T*>(ip.gather(ip.rank, par, c->s));
        }
    }
    bool finished = false;
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        const Slab& s = c->slabs[si];
        const Scalars<T>* gate = gated ? (gate_or_null ? gate_or_null : S[si]) : nullptr;
        TreePlan plan = s.plan;
        if (leaves && (*leaves)[si] > 0) {
            plan.blocks = (*leaves)[si];
        } else {
            launch_tree_stage1<T>(s.plan, static_cast<const T*>(s.part[0]),
                                  static_cast<const T*>(s.part[1]),
                                  static_cast<const T*>(s.part[2]), nv,
                                  static_cast<T*>(s.stage), gate, c->stream);
        }
        T* g = c->comm ? static_cast<T*>(c->gather_send) : gather;
        const int slot = c->comm ? 0 : s.index;
        finished = launch_tree_stage2<T>(plan, static_cast<const T*>(s.stage), nv, g, slot, single,
                                         c->nslabs_total, c->exact_tree, S[si], op, c->stream,
                                         put.n ? &put : nullptr);
    }
    if (single || finished) return;
    const unsigned long long* wait_flags = nullptr;
    if (c->ipc) {
        IpcState& ip = *c->ipc;
        wait_flags = ip.flags(ip.rank) + 2;
        gather = reinterpret_cast<T*>(ip.gather(ip.rank, par, c->s));
    } else if (c->comm) {
        const ncclDataType_t dt = c->dtype == ACG_F32 ? ncclFloat32 : ncclFloat64;
        nccl_comm_alive(c->comm);
        nccl_comm_check(c->comm,
                        nccl().allGather(c->gather_send, c->gather, 4, dt, c->comm->comm, c->stream),
                        "ncclAllGather");
    }
    for (size_t si = 0; si < c->slabs.size(); ++si)
        launch_finish<T>(gather, nv, c->nslabs_total, c->exact_tree, S[si], op, c->stream,
                         wait_flags, seq);
}

template <typename T>
std::vector<Scalars<T>*> tmp_scalars(const acg_context* c) {
    std::vector<Scalars<T>*> v;
    for (const Slab& s : c->slabs) v.push_back(static_cast<Scalars<T>*>(s.tmp));
    return v;
}

template <typename T>
Scalars<T> read_scalars(const acg_context* c, const Scalars<T>* dev) {
    Scalars<T> h;
    CK(cudaMemcpyAsync(&h, dev, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return h;
}

template <typename T>
void reset_tmp(const acg_context* c, T alpha = T(0), T beta = T(0)) {
    Scalars<T> h{};
    h.alpha = alpha;
    h.beta = beta;
    for (const Slab& s : c->slabs)
        CK(cudaMemcpyAsync(s.tmp, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
}

// ------------------------------------------------------------ device ops
template <typename T>
void op_apply(const acg_context* c, const acg_field* x, acg_field* y, const Scalars<T>* gate) {
    halo(c, x);
    for (size_t si = 0; si < c->slabs.size(); ++si)
        launch_apply<T>(view<T>(c, si), c->fast(), static_cast<const T*>(x->data(si)),
                        static_cast<T*>(y->data(si)), gate, c->stream);
}

template <typename T>
void op_precondition(const acg_context* c, const acg_field* y, acg_field* x,
                     const std::vector<Scalars<T>*>& flag, const Scalars<T>* gate) {
    for (size_t si = 0; si < c->slabs.size(); ++si)
        launch_precondition<T>(view<T>(c, si), c->fast(), static_cast<const T*>(y->data(si)),
                               static_cast<T*>(x->data(si)), flag[si], gate,
                               static_cast<T*>(c->slabs[si].phi), c->stream);
}

template <typename T>
void op_dot(const acg_context* c, const acg_field* x, const acg_field* y, int op,
            const std::vector<Scalars<T>*>& S, bool gated) {
    for (size_t si = 0; si < c->slabs.size(); ++si)
        launch_dot_partials<T>(view<T>(c, si), static_cast<const T*>(x->data(si)),
                               static_cast<const T*>(y->data(si)),
                               static_cast<T*>(c->slabs[si].part[0]), gated ? S[si] : nullptr,
                               c->stream);
    reduce<T>(c, 1, op, S, nullptr, gated);
}

template <typename T>
void op_axpy(const acg_context* c, T value, const std::vector<Scalars<T>*>* coefS, int which,
             bool neg, const acg_field* x, acg_field* y, bool gated) {
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        const T* coef = nullptr;
        const Scalars<T>* g = nullptr;
        if (coefS) {
            Scalars<T>* S = (*coefS)[si];
            coef = which == 0 ? &S->alpha : (which == 1 ? &S->beta : nullptr);
            if (gated) g = S;  // gated on the solver's done flag
        }
        launch_axpy<T>(c->slabs[si].n_loc, value, coef, neg, static_cast<const T*>(x->data(si)),
                       static_cast<T*>(y->data(si)), g, c->stream);
    }
}

template <typename T>
void op_copy(const acg_context* c, const acg_field* x, acg_field* y, const std::vector<Scalars<T>*>* gS) {
    for (size_t si = 0; si < c->slabs.size(); ++si)
        launch_copy<T>(c->slabs[si].n_loc, static_cast<const T*>(x->data(si)),
                       static_cast<T*>(y->data(si)), gS ? (*gS)[si] : nullptr, c->stream);
}

// ---------------------------------------------------- matrix-explicit backend
// CsrBackend (solver.hpp:126-145): the CSR matrix and the stored tridiagonals,
// assembled on the device the first time a solve asks for them (rows ordered
// for `layout`, csr.hpp:92-124) and kept until release_scratch.
template <typename T>
void ensure_csr(const acg_context* cc, int layout) {
    NvtxRange nr("acg csr assemble");
    acg_context* c = const_cast<acg_context*>(cc);
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        Slab& s = c->slabs[si];
        if (s.csr_layout == layout) continue;
        free_csr(s);
        if (s.n_loc + 2 * s.plane >= (1ll << 31))
            fail(ACG_ERR_INVALID_ARGUMENT,
                 "csr backend: %lld rows per slab exceed the 32-bit column index of CsrMatrix",
                 s.n_loc);
        const long long m = c->m, n_z = c->n_z;
        // nnz of the slab's planes: every row has itself plus its in-panel neighbours
        long long nnz = 0;
        for (int il = 0; il < s.m_loc; ++il) {
            const int i = s.i0 + il;
            const long long ci = (i > 0) + (i + 1 < m);
            nnz += n_z * m * (1 + ci) + n_z * (m > 1 ? 2 * (m - 1) : 0) +
                   m * (n_z > 1 ? 2 * (n_z - 1) : 0);
        }
        CK(cudaMalloc(&s.csr_rp, (s.n_loc + 1) * sizeof(long long)));
        CK(cudaMalloc(&s.csr_ci, nnz * sizeof(int)));
        CK(cudaMalloc(&s.csr_val, nnz * sizeof(T)));
        for (void*& t : s.tri) CK(cudaMalloc(&t, s.n_loc * sizeof(T)));
        CK(cudaMalloc(&s.tri_phi, s.n_loc * sizeof(T)));
        launch_csr_assemble<T>(view<T>(c, si), layout == ACG_LAYOUT_HORIZONTAL ? 1 : 0, s.csr_rp,
                               s.csr_ci, static_cast<T*>(s.csr_val), static_cast<T*>(s.tri[0]),
                               static_cast<T*>(s.tri[1]), static_cast<T*>(s.tri[2]), c->stream);
        CK(cudaPeekAtLastError());
        s.csr_layout = layout;
    }
}

// spmv_csr (csr.hpp:127-141)
template <typename T>
void op_spmv_csr(const acg_context* c, const acg_field* x, acg_field* y, const Scalars<T>* gate) {
    halo(c, x);
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        const Slab& s = c->slabs[si];
        launch_csr_spmv<T>(view<T>(c, si), s.csr_rp, s.csr_ci, static_cast<const T*>(s.csr_val),
                           static_cast<const T*>(x->data(si)), static_cast<T*>(y->data(si)), gate,
                           c->stream);
    }
}

// solve_tridiag_set (csr.hpp:175-221)
template <typename T>
void op_tridiag(const acg_context* c, const acg_field* y, acg_field* x,
                const std::vector<Scalars<T>*>& flag, const Scalars<T>* gate) {
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        const Slab& s = c->slabs[si];
        launch_csr_tridiag<T>(view<T>(c, si), static_cast<const T*>(s.tri[0]),
                              static_cast<const T*>(s.tri[1]), static_cast<const T*>(s.tri[2]),
                              static_cast<const T*>(y->data(si)), static_cast<T*>(x->data(si)),
                              static_cast<T*>(s.tri_phi), flag[si], gate, c->stream);
    }
}

template <typename T>
T op_true_residual(const acg_context* c, const acg_field* u, const acg_field* f) {
    halo(c, u);
    for (size_t si = 0; si < c->slabs.size(); ++si)
        launch_residual_partials<T>(view<T>(c, si), c->fast(), static_cast<const T*>(u->data(si)),
                                    static_cast<const T*>(f->data(si)),
                                    static_cast<T*>(c->slabs[si].part[0]), c->stream);
    auto S = tmp_scalars<T>(c);
    reset_tmp<T>(c);
    reduce<T>(c, 1, kOpStore, S, nullptr, false);
    const Scalars<T> h = read_scalars<T>(c, S[0]);
    return std::sqrt(h.val[0]);  // nrm2's sqrt in T (field.hpp:172)
}

// true_residual(CsrMatrix, u, f), solver.hpp:71-78: t = A u; t = -t; t += f; ||t||
template <typename T>
T op_true_residual_csr(const acg_context* c, const acg_field* u, const acg_field* f, acg_field* t) {
    op_spmv_csr<T>(c, u, t, nullptr);
    for (size_t si = 0; si < c->slabs.size(); ++si)
        launch_scal<T>(c->slabs[si].n_loc, T(-1), nullptr, static_cast<T*>(t->data(si)), nullptr,
                       c->stream);
    op_axpy<T>(c, T(1), nullptr, -1, false, f, t, false);
    auto S = tmp_scalars<T>(c);
    reset_tmp<T>(c);
    op_dot<T>(c, t, t, kOpStore, S, false);
    const Scalars<T> h = read_scalars<T>(c, S[0]);
    return std::sqrt(h.val[0]);
}

void check_same(const acg_field* a, const acg_field* b, const char* what) {
    if (!a || !b) fail(ACG_ERR_INVALID_ARGUMENT, "%s: null field", what);
    if (!a->ctx || !b->ctx) fail(ACG_ERR_INVALID_ARGUMENT, "%s: field of a destroyed context", what);
    if (a->ctx->m != b->ctx->m || a->ctx->n_z != b->ctx->n_z || a->ctx->dtype != b->ctx->dtype ||
        a->ctx->slabs.size() != b->ctx->slabs.size())
        fail(ACG_ERR_INVALID_ARGUMENT, "%s: shape/layout mismatch", what);
}

#define ACG_TDISPATCH(ctx, ...)          \
    do {                                 \
        if ((ctx)->dtype == ACG_F32) {   \
            using T = float;             \
            __VA_ARGS__;                 \
        } else {                         \
            using T = double;            \
            __VA_ARGS__;                 \
        }                                \
    } while (0)

}  // namespace

extern "C" {

acg_status acg_field_create(acg_field** out, const acg_context* c) {
    return guarded([&] {
        check_ctx(c);
        if (!out) fail(ACG_ERR_INVALID_ARGUMENT, "null output");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        *out = new_field(c);
        c->user_fields.push_back(*out);
    });
}

acg_status acg_field_destroy(acg_field* f) {
    return guarded([&] {
        if (!f) return;
        if (!f->ctx) {  // orphaned by acg_context_destroy: device memory already freed
            delete f;
            return;
        }
        const acg_context* c = f->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        auto& v = c->user_fields;
        v.erase(std::remove(v.begin(), v.end(), f), v.end());
        cudaStreamSynchronize(c->stream);
        free_field(f);
    });
}

acg_status acg_field_upload(acg_field* f, const void* host, acg_layout layout,
                            acg_host_scope scope) {
    return guarded([&] {
        if (!f || !host) fail(ACG_ERR_INVALID_ARGUMENT, "null argument");
        const acg_context* c = f->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        await_field(c, f);
        ACG_TDISPATCH(c, upload_t<T>(f, host, layout, scope));
    });
}

acg_status acg_field_download(const acg_field* f, void* host, acg_layout layout,
                              acg_host_scope scope) {
    return guarded([&] {
        if (!f || !host) fail(ACG_ERR_INVALID_ARGUMENT, "null argument");
        const acg_context* c = f->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        await_field(c, f);
        ACG_TDISPATCH(c, download_t<T>(f, host, layout, scope));
    });
}

acg_status acg_field_upload_async(acg_field* f, const void* host, acg_layout layout,
                                  acg_host_scope scope) {
    return guarded([&] {
        if (!f || !host) fail(ACG_ERR_INVALID_ARGUMENT, "null argument");
        const acg_context* c = f->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        ACG_TDISPATCH(c, upload_t<T>(f, host, layout, scope, true));
    });
}

acg_status acg_field_download_async(const acg_field* f, void* host, acg_layout layout,
                                    acg_host_scope scope) {
    return guarded([&] {
        if (!f || !host) fail(ACG_ERR_INVALID_ARGUMENT, "null argument");
        const acg_context* c = f->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        ACG_TDISPATCH(c, download_t<T>(f, host, layout, scope, true));
    });
}

acg_status acg_field_wait(const acg_field* f) {
    return guarded([&] {
        if (!f) fail(ACG_ERR_INVALID_ARGUMENT, "null field");
        const acg_context* c = f->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        if (f->ev) CK(cudaEventSynchronize(f->ev));
    });
}

acg_status acg_field_upload_device(acg_field* f, const void* dev, acg_layout layout,
                                   acg_host_scope scope) {
    return guarded([&] {
        if (!f || !dev) fail(ACG_ERR_INVALID_ARGUMENT, "null argument");
        const acg_context* c = f->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        await_field(c, f);
        ACG_TDISPATCH(c, upload_dev_t<T>(f, dev, layout, scope));
    });
}

acg_status acg_field_download_device(const acg_field* f, void* dev, acg_layout layout,
                                     acg_host_scope scope) {
    return guarded([&] {
        if (!f || !dev) fail(ACG_ERR_INVALID_ARGUMENT, "null argument");
        const acg_context* c = f->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        await_field(c, f);
        ACG_TDISPATCH(c, download_dev_t<T>(f, dev, layout, scope));
    });
}

acg_status acg_field_fill(acg_field* f, double value) {
    return guarded([&] {
        if (!f) fail(ACG_ERR_INVALID_ARGUMENT, "null field");
        const acg_context* c = f->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        await_field(c, f);
        ACG_TDISPATCH(c, {
            for (size_t si = 0; si < c->slabs.size(); ++si)
                launch_fill<T>(c->slabs[si].n_loc, static_cast<T>(value),
                               static_cast<T*>(f->data(si)), c->stream);
        });
        CK(cudaPeekAtLastError());
    });
}

acg_status acg_field_fill_random(acg_field* f, uint64_t seed) {
    return guarded([&] {
        if (!f) fail(ACG_ERR_INVALID_ARGUMENT, "null field");
        const acg_context* c = f->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        await_field(c, f);
        ACG_TDISPATCH(c, {
            for (size_t si = 0; si < c->slabs.size(); ++si)
                launch_fill_random<T>(view<T>(c, si), seed, static_cast<T*>(f->data(si)),
                                      c->stream);
        });
        CK(cudaPeekAtLastError());
    });
}

acg_status acg_field_copy(acg_field* dst, const acg_field* src) {
    return guarded([&] {
        check_same(dst, src, "copy");
        const acg_context* c = dst->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        await_field(c, dst);
        await_field(c, src);
        ACG_TDISPATCH(c, op_copy<T>(c, src, dst, nullptr));
        CK(cudaPeekAtLastError());
    });
}

acg_status acg_apply(const acg_context* c, const acg_field* x, acg_field* y) {
    return guarded([&] {
        check_ctx(c);
        check_field(c, x, "apply");
        check_field(c, y, "apply");
        if (x == y) fail(ACG_ERR_INVALID_ARGUMENT, "apply: x and y must not alias");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        ACG_TDISPATCH(c, op_apply<T>(c, x, y, nullptr));
        CK(cudaPeekAtLastError());
    });
}

acg_status acg_precondition(const acg_context* c, const acg_field* y, acg_field* x) {
    return guarded([&] {
        check_ctx(c);
        check_field(c, y, "precondition");
        check_field(c, x, "precondition");
        if (x == y) fail(ACG_ERR_INVALID_ARGUMENT, "precondition: y and x must not alias");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        ACG_TDISPATCH(c, {
            reset_tmp<T>(c);
            auto S = tmp_scalars<T>(c);
            op_precondition<T>(c, y, x, S, nullptr);
            CK(cudaPeekAtLastError());
            for (Scalars<T>* s : S)
                if (read_scalars<T>(c, s).pivot)
                    fail(ACG_ERR_BREAKDOWN, "precondition: zero pivot in tridiagonal elimination");
        });
    });
}

acg_status acg_axpy(double alpha, const acg_field* x, acg_field* y) {
    return guarded([&] {
        check_same(x, y, "axpy");
        const acg_context* c = x->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        await_field(c, x);
        await_field(c, y);
        ACG_TDISPATCH(c, op_axpy<T>(c, static_cast<T>(alpha), nullptr, -1, false, x, y, false));
        CK(cudaPeekAtLastError());
    });
}

acg_status acg_scal(double alpha, acg_field* x) {
    return guarded([&] {
        if (!x) fail(ACG_ERR_INVALID_ARGUMENT, "scal: null field");
        const acg_context* c = x->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        await_field(c, x);
        ACG_TDISPATCH(c, {
            for (size_t si = 0; si < c->slabs.size(); ++si)
                launch_scal<T>(c->slabs[si].n_loc, static_cast<T>(alpha), nullptr,
                               static_cast<T*>(x->data(si)), nullptr, c->stream);
        });
        CK(cudaPeekAtLastError());
    });
}

acg_status acg_dot(const acg_field* x, const acg_field* y, double* out) {
    return guarded([&] {
        check_same(x, y, "dot");
        if (!out) fail(ACG_ERR_INVALID_ARGUMENT, "null output");
        const acg_context* c = x->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        await_field(c, x);
        await_field(c, y);
        ACG_TDISPATCH(c, {
            reset_tmp<T>(c);
            auto S = tmp_scalars<T>(c);
            op_dot<T>(c, x, y, kOpStore, S, false);
            *out = static_cast<double>(read_scalars<T>(c, S[0]).val[0]);
        });
    });
}

acg_status acg_nrm2(const acg_field* x, double* out) {
    return guarded([&] {
        if (!x || !out) fail(ACG_ERR_INVALID_ARGUMENT, "null argument");
        const acg_context* c = x->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "field of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        await_field(c, x);
        ACG_TDISPATCH(c, {
            reset_tmp<T>(c);
            auto S = tmp_scalars<T>(c);
            op_dot<T>(c, x, x, kOpStore, S, false);
            *out = static_cast<double>(std::sqrt(read_scalars<T>(c, S[0]).val[0]));
        });
    });
}

acg_status acg_true_residual(const acg_context* c, const acg_field* u, const acg_field* f,
                             double* out) {
    return guarded([&] {
        check_ctx(c);
        check_field(c, u, "true_residual");
        check_field(c, f, "true_residual");
        if (!out) fail(ACG_ERR_INVALID_ARGUMENT, "null output");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        ACG_TDISPATCH(c, *out = static_cast<double>(op_true_residual<T>(c, u, f)));
    });
}

acg_status acg_interleaved_spmv_kernel(const acg_context* c, acg_field* u, acg_field* p,
                                       acg_field* q, const acg_field* z, double alpha,
                                       double beta, double* sigma) {
    return guarded([&] {
        check_ctx(c);
        for (const acg_field* f : {static_cast<const acg_field*>(u), static_cast<const acg_field*>(p),
                                   static_cast<const acg_field*>(q), z})
            check_field(c, f, "interleaved_spmv_kernel");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        ACG_TDISPATCH(c, {
            reset_tmp<T>(c, static_cast<T>(alpha), static_cast<T>(beta));
            auto S = tmp_scalars<T>(c);
            halo(c, z);
            std::vector<int> leaves(c->slabs.size());
            for (size_t si = 0; si < c->slabs.size(); ++si)
                leaves[si] = launch_fused_spmv<T>(
                    view<T>(c, si), c->fast(), static_cast<T*>(u->data(si)),
                    static_cast<T*>(p->data(si)), static_cast<T*>(q->data(si)),
                    static_cast<const T*>(z->data(si)), static_cast<T*>(c->slabs[si].part[0]),
                    S[si], static_cast<T*>(c->slabs[si].stage), c->stream);
            reduce<T>(c, 1, kOpStore, S, nullptr, false, &leaves);
            const Scalars<T> h = read_scalars<T>(c, S[0]);
            if (sigma) *sigma = static_cast<double>(h.val[0]);
        });
    });
}

acg_status acg_interleaved_prec_kernel(const acg_context* c, acg_field* r, acg_field* z,
                                       const acg_field* q, double alpha, double* r_norm,
                                       double* kappa) {
    return guarded([&] {
        check_ctx(c);
        for (const acg_field* f :
             {static_cast<const acg_field*>(r), static_cast<const acg_field*>(z), q})
            check_field(c, f, "interleaved_prec_kernel");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        ACG_TDISPATCH(c, {
            reset_tmp<T>(c, static_cast<T>(alpha));
            auto S = tmp_scalars<T>(c);
            std::vector<int> leaves(c->slabs.size());
            for (size_t si = 0; si < c->slabs.size(); ++si) {
                const Slab& s = c->slabs[si];
                leaves[si] = launch_fused_prec<T>(
                    view<T>(c, si), c->fast(), static_cast<T*>(r->data(si)),
                    static_cast<T*>(z->data(si)), static_cast<const T*>(q->data(si)),
                    static_cast<T*>(s.part[0]), static_cast<T*>(s.part[1]), S[si],
                    static_cast<T*>(s.phi), static_cast<T*>(s.stage), c->stream);
            }
            for (Scalars<T>* s : S)
                if (read_scalars<T>(c, s).pivot)
                    fail(ACG_ERR_BREAKDOWN,
                         "interleaved_prec_kernel: zero pivot in tridiagonal elimination");
            reduce<T>(c, 2, kOpStore, S, nullptr, false, &leaves);
            const Scalars<T> h = read_scalars<T>(c, S[0]);
            if (r_norm) *r_norm = static_cast<double>(std::sqrt(h.val[0]));
            if (kappa) *kappa = static_cast<double>(h.val[1]);
        });
    });
}

void acg_solve_result_release(acg_solve_result* res) {
    if (!res) return;
    for (double*& h : res->history) {
        std::free(h);
        h = nullptr;
    }
}

void acg_solver_config_default(acg_solver_config* cfg) {
    if (!cfg) return;
    cfg->epsilon = 1e-5;
    cfg->tau = 1e-20;
    cfg->maxiter = 500;
    cfg->variant = ACG_VARIANT_STANDARD;  // SolverConfig default (solver.hpp:23)
    cfg->backend = ACG_BACKEND_MATRIX_FREE;
    cfg->workers = 1;
    cfg->record_timings = 0;
    cfg->layout = ACG_LAYOUT_VERTICAL;
}

}  // extern "C"

// ==================================================================== solver
namespace {

enum Family { kSpmv = 0, kPrec, kBlas, kFusedSpmv, kFusedPrec, kFamilies };

struct EventTimer {
    bool on = false;
    cudaStream_t st = nullptr;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<std::pair<size_t, size_t>> marks[kFamilies];
    size_t open_idx = 0;
    cudaEvent_t next() {
        if (used == pool.size()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return pool[used++];
    }
    void begin(int) {
        if (!on) return;
        open_idx = used;
        CK(cudaEventRecord(next(), st));
    }
    void end(int fam) {
        if (!on) return;
        const size_t b = open_idx;
        CK(cudaEventRecord(next(), st));
        marks[fam].emplace_back(b, used - 1);
    }
    double seconds(int fam) {
        double ms = 0;
        for (auto& pr : marks[fam]) {
            float t = 0;
            CK(cudaEventElapsedTime(&t, pool[pr.first], pool[pr.second]));
            ms += t;
        }
        return ms * 1e-3;
    }
    int count(int fam) const { return static_cast<int>(marks[fam].size()); }
    void reset() {
        used = 0;
        for (auto& m : marks) m.clear();
    }
    ~EventTimer() { release(); }
    void release() {
        for (cudaEvent_t e : pool) cudaEventDestroy(e);
        pool.clear();
        used = 0;
        for (auto& mk : marks) mk.clear();
    }
};

}  // namespace

struct acg_solver {
    const acg_context* ctx = nullptr;
    acg_solver_config cfg{};
    acg_field *u = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
    const acg_field* f = nullptr;
    std::vector<void*> S;     // Scalars<T>* per local slab
    std::vector<double*> hist;  // 4 arrays per local slab
    void* mirror = nullptr;   // pinned 2 x Scalars<T>, mapped
    void* mirror_dev = nullptr;  // its device address (launch_snapshot target)
    cudaEvent_t mev[2] = {nullptr, nullptr};
    bool started = false;
    int cap = 0;              // device history ring capacity (entries, power of two)
    std::vector<double> hv[4];  // host copies of the histories (drained from the rings)
    int drained[4] = {0, 0, 0, 0};
    int undrained = 0;          // step API: iterations enqueued since the last drain
    long long launches0 = 0;
    EventTimer timer;       // per-family timings (record_timings)
    EventTimer ktimer;      // per-launch timing of K1/K2 (bench)
    std::vector<int> leaves;  // per slab: tree leaves the last sweep wrote (fused stage 1)
    // consumed-reduction mode (Consume, acg_internal.h): the second state buffer
    // (K1 writes it, K2 reads it) and the K2 leaves whose finish is pending
    void* S_alt = nullptr;
    bool consume_pending = false;
    int consume_leaves = 0;
    bool csr = false;         // matrix-explicit backend (standard loop on CSR + tridiagonals)
    // CUDA graph of kGraphChunk iterations (single-process contexts, small grids):
    // replayed instead of re-launching the same kernels every iteration
    cudaGraphExec_t chunk = nullptr;
    long long chunk_launches = 0;  // kernels per replay (for the launch counter)
    bool chunk_failed = false;
    int chunk_kind = -1;           // variant * 2 + csr the graph was captured for
    std::chrono::steady_clock::time_point t0;
    double setup_s = 0.0;
    ~acg_solver() { release(); }
    void release() {  // device resources; idempotent
        if (chunk) cudaGraphExecDestroy(chunk);
        chunk = nullptr;
        for (acg_field** fl : {&u, &r, &z, &p, &q}) {
            if (*fl) free_field(*fl);
            *fl = nullptr;
        }
        for (void* s : S) cudaFree(s);
        S.clear();
        if (S_alt) cudaFree(S_alt);
        S_alt = nullptr;
        for (double* h : hist) cudaFree(h);
        hist.clear();
        if (mirror) cudaFreeHost(mirror);
        mirror = nullptr;
        for (cudaEvent_t& e : mev) {
            if (e) cudaEventDestroy(e);
            e = nullptr;
        }
        timer.release();
        ktimer.release();
    }
};

void orphan_solver(acg_solver* s) {
    s->release();
    s->ctx = nullptr;
}

void destroy_cached_solver(acg_context* c) {
    delete c->cached;
    c->cached = nullptr;
}

namespace {

void validate(const acg_solver_config* cfg) {
    if (!cfg) fail(ACG_ERR_INVALID_ARGUMENT, "null config");
    // SolverConfig::validate, solver.hpp:27-35
    if (!(cfg->epsilon > 0.0)) fail(ACG_ERR_INVALID_ARGUMENT, "SolverConfig: epsilon must be > 0");
    if (!(cfg->tau > 0.0)) fail(ACG_ERR_INVALID_ARGUMENT, "SolverConfig: tau must be > 0");
    if (cfg->maxiter < 1) fail(ACG_ERR_INVALID_ARGUMENT, "SolverConfig: maxiter must be >= 1");
    if (cfg->workers < 1) fail(ACG_ERR_INVALID_ARGUMENT, "SolverConfig: workers must be >= 1");
    if (cfg->variant == ACG_VARIANT_INTERLEAVED && cfg->backend == ACG_BACKEND_CSR)
        fail(ACG_ERR_INVALID_ARGUMENT,
             "SolverConfig: the interleaved variant exists for the matrix-free backend only");
    if (cfg->backend != ACG_BACKEND_MATRIX_FREE && cfg->backend != ACG_BACKEND_CSR)
        fail(ACG_ERR_INVALID_ARGUMENT, "SolverConfig: unknown backend");
    if (cfg->variant != ACG_VARIANT_STANDARD && cfg->variant != ACG_VARIANT_INTERLEAVED)
        fail(ACG_ERR_INVALID_ARGUMENT, "SolverConfig: unknown variant");
    if (cfg->layout != ACG_LAYOUT_VERTICAL && cfg->layout != ACG_LAYOUT_HORIZONTAL)
        fail(ACG_ERR_INVALID_ARGUMENT, "SolverConfig: unknown layout");
}

template <typename T>
std::vector<Scalars<T>*> sv(acg_solver* s) {
    std::vector<Scalars<T>*> v;
    for (void* p : s->S) v.push_back(static_cast<Scalars<T>*>(p));
    return v;
}

template <typename T>
void solver_alloc(acg_solver* s) {
    const acg_context* c = s->ctx;
    const int cap = kHistRing;  // independent of maxiter: the host drains the rings
    s->cap = cap;
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        void* p = nullptr;
        CK(cudaMalloc(&p, sizeof(Scalars<T>)));
        s->S.push_back(p);
        for (int a = 0; a < 4; ++a) {
            double* h = nullptr;
            CK(cudaMalloc(&h, cap * sizeof(double)));
            s->hist.push_back(h);
        }
    }
    if (c->slabs.size() == 1) CK(cudaMalloc(&s->S_alt, sizeof(Scalars<T>)));
    CK(cudaHostAlloc(&s->mirror, 2 * sizeof(Scalars<T>), cudaHostAllocPortable | cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&s->mirror_dev, s->mirror, 0));
    for (auto& e : s->mev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    s->u = new_field(c, false);
    s->r = new_field(c, false);
    s->z = new_field(c, false);
    s->p = new_field(c, false);
    s->q = new_field(c, false);
}

// Solver state cached in the context between solve calls (the five work
// fields alone are 5 x N x s bytes; re-allocating them per call dominated the
// end-to-end time of repeated solves).
template <typename T>
acg_solver* cached_solver(const acg_context* c, const acg_solver_config* cfg) {
    acg_context* cc = const_cast<acg_context*>(c);
    if (!cc->cached) {
        auto s = std::make_unique<acg_solver>();
        s->ctx = c;
        s->cfg = *cfg;
        solver_alloc<T>(s.get());
        cc->cached = s.release();
    }
    cc->cached->cfg = *cfg;
    cc->cached->started = false;
    return cc->cached;
}

template <typename T>
void solver_start(acg_solver* s, const acg_field* f, const acg_field* u0) {
    NvtxRange nr("acg solve init");
    const acg_context* c = s->ctx;
    s->t0 = std::chrono::steady_clock::now();
    s->launches0 = g_launches.load();
    s->f = f;
    s->csr = s->cfg.backend == ACG_BACKEND_CSR;
    if (s->csr) {  // make_backend (solver.hpp:147-154): assembly counts as setup
        const auto t = std::chrono::steady_clock::now();
        ensure_csr<T>(c, s->cfg.layout);
        CK(cudaStreamSynchronize(c->stream));
        s->setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
    } else {
        s->setup_s = 0.0;
    }
    for (int a = 0; a < 4; ++a) {
        s->hv[a].clear();
        s->drained[a] = 0;
    }
    s->undrained = 0;
    s->timer.st = c->stream;
    s->ktimer.st = c->stream;
    s->timer.on = s->cfg.record_timings != 0;
    s->timer.reset();
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        Scalars<T> h{};
        h.eps = s->cfg.epsilon;
        h.tau = s->cfg.tau;
        h.maxiter = s->cfg.maxiter;
        h.it = 1;
        h.hmask = s->cap - 1;
        h.h_res = s->hist[si * 4 + 0];
        h.h_kap = s->hist[si * 4 + 1];
        h.h_alp = s->hist[si * 4 + 2];
        h.h_bet = s->hist[si * 4 + 3];
        CK(cudaMemcpyAsync(s->S[si], &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
    }
    auto S = sv<T>(s);
    // u = u0, r = f (solver.hpp:288-290)
    if (u0)
        op_copy<T>(c, u0, s->u, nullptr);
    else
        for (size_t si = 0; si < c->slabs.size(); ++si)
            launch_fill<T>(c->slabs[si].n_loc, T(0), static_cast<T*>(s->u->data(si)), c->stream);
    op_copy<T>(c, f, s->r, nullptr);
    // q = A u; r = r - q; ||r0||  (:295-305)
    s->timer.begin(kSpmv);
    if (s->csr)
        op_spmv_csr<T>(c, s->u, s->q, S[0]);
    else
        op_apply<T>(c, s->u, s->q, S[0]);
    s->timer.end(kSpmv);
    s->timer.begin(kBlas);
    op_axpy<T>(c, T(-1), nullptr, -1, false, s->q, s->r, false);
    op_dot<T>(c, s->r, s->r, kOpR0, S, true);
    s->timer.end(kBlas);
    // z = M^-1 r; kappa_old = <r,z>  (:313-323)
    s->timer.begin(kPrec);
    if (s->csr)
        op_tridiag<T>(c, s->r, s->z, S, S[0]);
    else
        op_precondition<T>(c, s->r, s->z, S, S[0]);
    s->timer.end(kPrec);
    s->timer.begin(kBlas);
    op_dot<T>(c, s->r, s->z, kOpKappa0, S, true);
    s->timer.end(kBlas);
    // p = z
    op_copy<T>(c, s->z, s->p, &S);
    if (s->cfg.variant == ACG_VARIANT_INTERLEAVED) {
        // q = A p; sigma = <p,q>; alpha  (:325-336)
        s->timer.begin(kSpmv);
        op_apply<T>(c, s->p, s->q, S[0]);
        s->timer.end(kSpmv);
        s->timer.begin(kBlas);
        op_dot<T>(c, s->p, s->q, kOpSigma0, S, true);
        s->timer.end(kBlas);
    }
    CK(cudaPeekAtLastError());
    s->started = true;
}

// Consumed-reduction mode for this solver's loop (single slab in one process,
// both sweeps the fused-reduction kernels with few leaves: small grids).
template <typename T>
bool consume_mode(const acg_solver* s, int* l1, int* l2) {
    const acg_context* c = s->ctx;
    if (s->S_alt == nullptr || c->slabs.size() != 1 || c->nslabs_total != 1 || c->ipc || c->comm)
        return false;
    return consume_plan<T>(view<T>(c, 0), c->slabs[0].phi != nullptr, l1, l2);
}

// The last K2's pending reduction finish (kOpIlSpmv on state A): one tree kernel
// at the end of a batch, after which S[0] holds the complete state again.
template <typename T>
void consume_flush(acg_solver* s) {
    if (!s->consume_pending) return;
    const acg_context* c = s->ctx;
    TreePlan plan{};
    plan.blocks = s->consume_leaves;
    launch_tree_stage2<T>(plan, static_cast<const T*>(c->slabs[0].stage) + kConsumeK2Stage, 1,
                          static_cast<T*>(c->gather), 0, true, 1, c->exact_tree,
                          static_cast<Scalars<T>*>(s->S[0]), kOpIlSpmv, c->stream, nullptr);
    s->consume_pending = false;
}

// One interleaved iteration in consumed-reduction mode: K1 finishes the previous
// K2's reduction in its prologue (state A -> B), K2 finishes K1's (B -> A).
template <typename T>
void iterate_interleaved_consumed(acg_solver* s, int l1, int l2) {
    const acg_context* c = s->ctx;
    const Slab& sl = c->slabs[0];
    T* stage = static_cast<T*>(sl.stage);
    Scalars<T>* A = static_cast<Scalars<T>*>(s->S[0]);
    Scalars<T>* B = static_cast<Scalars<T>*>(s->S_alt);
    const Consume<T> c1{stage + kConsumeK2Stage, l2, 1, kOpIlSpmv, A, B};
    const Consume<T> c2{stage, l1, 2, kOpIlPrec, B, A};
    const SlabView<T> v = view<T>(c, 0);
    s->timer.begin(kFusedPrec);
    s->ktimer.begin(kFusedPrec);
    launch_fused_prec<T>(v, c->fast(), static_cast<T*>(s->r->data(0)),
                         static_cast<T*>(s->z->data(0)), static_cast<const T*>(s->q->data(0)),
                         static_cast<T*>(sl.part[0]), static_cast<T*>(sl.part[1]), A, nullptr,
                         stage, c->stream, &c1);
    s->ktimer.end(kFusedPrec);
    s->timer.end(kFusedPrec);
    s->timer.begin(kFusedSpmv);
    s->ktimer.begin(kFusedSpmv);
    launch_fused_spmv<T>(v, c->fast(), static_cast<T*>(s->u->data(0)),
                         static_cast<T*>(s->p->data(0)), static_cast<T*>(s->q->data(0)),
                         static_cast<const T*>(s->z->data(0)), static_cast<T*>(sl.part[0]), B,
                         stage + kConsumeK2Stage, c->stream, &c2);
    s->ktimer.end(kFusedSpmv);
    s->timer.end(kFusedSpmv);
    s->consume_pending = true;
    s->consume_leaves = l2;
}

// One iteration of the interleaved loop (solver.hpp:338-365): two sweeps,
// two reductions, all gated on the device-side `done` flag.
template <typename T>
void iterate_interleaved(acg_solver* s) {
    const acg_context* c = s->ctx;
    int l1 = 0, l2 = 0;
    if (consume_mode<T>(s, &l1, &l2)) {
        iterate_interleaved_consumed<T>(s, l1, l2);
        return;
    }
    auto S = sv<T>(s);
    std::vector<int>& leaves = s->leaves;
    leaves.resize(c->slabs.size());
    // Peer-memory halo fused into the sweeps: K1 stores its boundary
    // planes into the neighbours' mailboxes and releases their flags; K2's boundary
    // CTAs acquire them and read the ghost rows from the local mailbox. No copy or
    // signal launches, no second stream.
    HaloLink<T> hl;
    if (c->ipc && c->slabs.size() == 1 &&
        fused_halo_ok<T>(view<T>(c, 0), c->fast(), c->slabs[0].phi != nullptr)) {
        IpcState& ip = *c->ipc;
        const int r = ip.rank, p = ip.p;
        const unsigned long long seq = ++ip.halo_seq;
        const int par = static_cast<int>(seq & 1);
        hl.on = 1;
        hl.seq = seq;
        hl.arrive = ip.arrive;
        if (r > 0) {  // plane 0 <-> rank r-1 (its ghost "from above"; mine "from below")
            hl.put[0] = reinterpret_cast<T*>(ip.ghost(r - 1, par, 1));
            hl.put_flag[0] = ip.flags(r - 1) + 1;
            hl.ghost[0] = reinterpret_cast<const T*>(ip.ghost(r, par, 0));
            hl.wait_flag[0] = ip.flags(r) + 0;
        }
        if (r + 1 < p) {  // plane m_loc-1 <-> rank r+1
            hl.put[1] = reinterpret_cast<T*>(ip.ghost(r + 1, par, 0));
            hl.put_flag[1] = ip.flags(r + 1) + 0;
            hl.ghost[1] = reinterpret_cast<const T*>(ip.ghost(r, par, 1));
            hl.wait_flag[1] = ip.flags(r) + 1;
        }
    }
    s->timer.begin(kFusedPrec);
    for (size_t si = 0; si < c->slabs.size(); ++si) {
        const Slab& sl = c->slabs[si];
        SlabView<T> v1 = view<T>(c, si);
        v1.halo = hl;
        s->ktimer.begin(kFusedPrec);
        leaves[si] = launch_fused_prec<T>(
            v1, c->fast(), static_cast<T*>(s->r->data(si)),
            static_cast<T*>(s->z->data(si)), static_cast<const T*>(s->q->data(si)),
            static_cast<T*>(sl.part[0]), static_cast<T*>(sl.part[1]), S[si],
            static_cast<T*>(sl.phi), static_cast<T*>(sl.stage), c->stream);
        s->ktimer.end(kFusedPrec);
    }
    reduce<T>(c, 2, kOpIlPrec, S, nullptr, true, &leaves);
    s->timer.end(kFusedPrec);
    s->timer.begin(kFusedSpmv);
    auto spmv = [&](size_t si, int pb, int pc) {
        SlabView<T> v = view<T>(c, si);
        v.plane_begin = pb;
        v.plane_count = pc;
        v.halo = hl;
        return launch_fused_spmv<T>(
            v, c->fast(), static_cast<T*>(s->u->data(si)), static_cast<T*>(s->p->data(si)),
            static_cast<T*>(s->q->data(si)), static_cast<const T*>(s->z->data(si)),
            static_cast<T*>(c->slabs[si].part[0]), S[si], static_cast<T*>(c->slabs[si].stage),
            c->stream);
    };
    const int m_loc0 = c->slabs[0].m_loc;
    if (hl.on) {
        s->ktimer.begin(kFusedSpmv);
        leaves[0] = spmv(0, 0, 0);
        s->ktimer.end(kFusedSpmv);
    } else if (c->halo_stream && m_loc0 >= 3 &&
        spmv_plane_ranges<T>(view<T>(c, 0), c->fast())) {
        // ranks > 1: the ghost planes travel on the halo stream while the interior
        // planes (which never read a ghost) are swept; the two boundary planes follow
        CK(cudaEventRecord(c->ev_ready, c->stream));
        CK(cudaStreamWaitEvent(c->halo_stream, c->ev_ready, 0));
        halo(c, s->z, c->halo_stream);
        CK(cudaEventRecord(c->ev_halo, c->halo_stream));
        s->ktimer.begin(kFusedSpmv);
        leaves[0] = spmv(0, 1, m_loc0 - 2);
        CK(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
        spmv(0, 0, 1);
        spmv(0, m_loc0 - 1, 1);
        s->ktimer.end(kFusedSpmv);
    } else {
        halo(c, s->z);
        for (size_t si = 0; si < c->slabs.size(); ++si) {
            s->ktimer.begin(kFusedSpmv);
            leaves[si] = spmv(si, 0, 0);
            s->ktimer.end(kFusedSpmv);
        }
    }
    reduce<T>(c, 1, kOpIlSpmv, S, nullptr, true, &leaves);
    s->timer.end(kFusedSpmv);
}

// One iteration of the standard loop (solver.hpp:217-262): 9 sweeps.
template <typename T>
void iterate_standard(acg_solver* s) {
    const acg_context* c = s->ctx;
    auto S = sv<T>(s);
    s->timer.begin(kSpmv);
    if (s->csr)
        op_spmv_csr<T>(c, s->p, s->q, S[0]);
    else
        op_apply<T>(c, s->p, s->q, S[0]);
    s->timer.end(kSpmv);
    s->timer.begin(kBlas);
    op_dot<T>(c, s->p, s->q, kOpStdSigma, S, true);
    op_axpy<T>(c, T(0), &S, 0, false, s->p, s->u, true);  // u = alpha p + u
    op_axpy<T>(c, T(0), &S, 0, true, s->q, s->r, true);   // r = (-alpha) q + r
    op_dot<T>(c, s->r, s->r, kOpStdRnorm, S, true);
    s->timer.end(kBlas);
    s->timer.begin(kPrec);
    if (s->csr)
        op_tridiag<T>(c, s->r, s->z, S, S[0]);
    else
        op_precondition<T>(c, s->r, s->z, S, S[0]);
    s->timer.end(kPrec);
    s->timer.begin(kBlas);
    op_dot<T>(c, s->r, s->z, kOpStdKappa, S, true);
    for (size_t si = 0; si < c->slabs.size(); ++si)  // p = beta p
        launch_scal<T>(c->slabs[si].n_loc, T(0), &S[si]->beta, static_cast<T*>(s->p->data(si)),
                       S[si], c->stream);
    op_axpy<T>(c, T(1), &S, -1, false, s->z, s->p, true);  // p = 1 z + p
    s->timer.end(kBlas);
}

template <typename T>
void solver_iterate_direct(acg_solver* s, int n) {
    for (int it = 0; it < n; ++it) {
        if (s->cfg.variant == ACG_VARIANT_INTERLEAVED)
            iterate_interleaved<T>(s);
        else
            iterate_standard<T>(s);
    }
    consume_flush<T>(s);
    CK(cudaPeekAtLastError());
}

constexpr int kGraphChunk = 16;

double bytes_per_iteration(const acg_context* c);

// Small grids replay a CUDA graph of kGraphChunk iterations instead of
// launching 4-5 kernels per iteration from the host: C1 (128^2 x 64) 45.1 ->
// 41.6 us per iteration; no change at C2/C3 (an A/B switch, since removed), so
// graphs are used below ~80 us of HBM traffic per iteration. Replay applies
// where every launch of an iteration is the same from one iteration to the
// next: one process (the peer-memory and NCCL transports put per-iteration
// sequence numbers into kernel arguments) and no per-launch event timers.
bool graph_wanted(const acg_solver* s) {
    return !s->chunk_failed && s->ctx->comm == nullptr && !s->timer.on && !s->ktimer.on &&
           bytes_per_iteration(s->ctx) < 0.5e9;
}

template <typename T>
bool build_chunk(acg_solver* s) {
    const acg_context* c = s->ctx;
    cudaGraph_t g = nullptr;
    const long long l0 = g_launches.load();
    if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    bool ok = true;
    try {
        solver_iterate_direct<T>(s, kGraphChunk);
    } catch (const Fail&) {
        ok = false;
    }
    const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (!ok || e != cudaSuccess || !g) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        g_launches -= g_launches.load() - l0;
        return false;
    }
    const cudaError_t ei = cudaGraphInstantiate(&s->chunk, g, 0);
    cudaGraphDestroy(g);
    s->chunk_launches = g_launches.load() - l0;
    g_launches -= s->chunk_launches;  // counted per replay instead
    if (ei != cudaSuccess) {
        cudaGetLastError();
        s->chunk = nullptr;
        return false;
    }
    return true;
}

template <typename T>
void solver_iterate(acg_solver* s, int n) {
    if (n >= kGraphChunk && graph_wanted(s)) {
        const int kind = s->cfg.variant * 2 + (s->csr ? 1 : 0);
        if (s->chunk && s->chunk_kind != kind) {  // a cached solver reused for another loop
            cudaGraphExecDestroy(s->chunk);
            s->chunk = nullptr;
        }
        if (!s->chunk) {
            if (build_chunk<T>(s))
                s->chunk_kind = kind;
            else
                s->chunk_failed = true;
        }
        if (s->chunk) {
            for (; n >= kGraphChunk; n -= kGraphChunk) {
                CK(cudaGraphLaunch(s->chunk, s->ctx->stream));
                g_launches += s->chunk_launches;
            }
        }
    }
    solver_iterate_direct<T>(s, n);
}

double bytes_per_iteration(const acg_context* c) {
    const double n = static_cast<double>(c->m) * c->m * c->n_z;
    return static_cast<double>(c->s) * (11.0 * n) / c->nslabs_total;
}

// Copy history entries [drained, counts) out of the device rings into the
// host vectors (synchronous). Entries written after `counts` stay in the ring:
// the caller drains before the device can be a full ring ahead.
void drain_histories(acg_solver* s, const int counts[4]) {
    const acg_context* c = s->ctx;
    const int cap = s->cap;
    for (int a = 0; a < 4; ++a) {
        const int lo = s->drained[a], hi = counts[a];
        if (hi <= lo) continue;
        if (hi - lo > cap) fail(ACG_ERR_INTERNAL, "history ring overrun (%d entries)", hi - lo);
        s->hv[a].resize(static_cast<size_t>(hi));
        int k = lo;
        while (k < hi) {  // at most two contiguous ring segments
            const int off = k & (cap - 1);
            const int n = std::min(hi - k, cap - off);
            CK(cudaMemcpyAsync(s->hv[a].data() + k, s->hist[a] + off, n * sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream));
            k += n;
        }
        s->drained[a] = hi;
    }
    CK(cudaStreamSynchronize(c->stream));
}

// Step API: enqueue n iterations; every half ring of iterations the stream is
// synchronised once and the history rings are drained (one short host stall
// per 2048 iterations), so any number of iterate() calls keeps every entry.
template <typename T>
void solver_iterate_drained(acg_solver* s, int n) {
    const int half = s->cap / 2;
    while (n > 0) {
        const int k = std::min(n, half - s->undrained);
        solver_iterate<T>(s, k);
        n -= k;
        s->undrained += k;
        if (s->undrained >= half) {
            const Scalars<T> h = read_scalars<T>(s->ctx, static_cast<Scalars<T>*>(s->S[0]));
            const int counts[4] = {h.n_res, h.n_kap, h.n_alp, h.n_bet};
            drain_histories(s, counts);
            s->undrained = 0;
        }
    }
}

// Enqueue iterations in batches; poll the done flag of the batch before the
// current one (pipelined, so the GPU never idles on the host).
template <typename T>
void solver_run(acg_solver* s) {
    NvtxRange nr("acg iterations");
    const acg_context* c = s->ctx;
    const double est_us = std::max(2.0, bytes_per_iteration(c) / 4.0e3);
    int batch = static_cast<int>(std::ceil(1500.0 / est_us));
    batch = std::max(1, std::min(batch, 64));
    Scalars<T>* mir = static_cast<Scalars<T>*>(s->mirror);
    Scalars<T>* mir_dev = static_cast<Scalars<T>*>(s->mirror_dev);
    constexpr int kWords = static_cast<int>(sizeof(Scalars<T>) / 8);
    int enq = 0, b = 0;
    // state after init (snapshots by a kernel: a D2H copy here would sit in the
    // copy engines' queue behind any asynchronous field transfer and hold the
    // solver's stream)
    launch_snapshot(s->S[0], &mir_dev[1], kWords, c->stream);
    CK(cudaEventRecord(s->mev[1], c->stream));
    CK(cudaEventSynchronize(s->mev[1]));
    if (mir[1].done) return;
    while (enq < s->cfg.maxiter) {
        const int n = std::min(batch, s->cfg.maxiter - enq);
        solver_iterate<T>(s, n);
        enq += n;
        launch_snapshot(s->S[0], &mir_dev[b & 1], kWords, c->stream);
        CK(cudaEventRecord(s->mev[b & 1], c->stream));
        if (b > 0) {
            CK(cudaEventSynchronize(s->mev[(b - 1) & 1]));
            const Scalars<T>& m = mir[(b - 1) & 1];
            if (m.done) break;
            // the device runs at most two batches (<= 128 entries per history)
            // ahead of this snapshot: drain well before a ring can wrap onto
            // undrained entries
            const int counts[4] = {m.n_res, m.n_kap, m.n_alp, m.n_bet};
            int most = 0;
            for (int a = 0; a < 4; ++a) most = std::max(most, counts[a] - s->drained[a]);
            if (most >= s->cap / 2) drain_histories(s, counts);
        }
        ++b;
    }
    CK(cudaStreamSynchronize(c->stream));
}

template <typename T>
void solver_finish(acg_solver* s, acg_field* u_out, acg_solve_result* res, double* hr, double* hk,
                   double* ha, double* hb) {
    NvtxRange nr("acg solve finish");
    const acg_context* c = s->ctx;
    auto S = sv<T>(s);
    CK(cudaStreamSynchronize(c->stream));
    Scalars<T> h = read_scalars<T>(c, S[0]);
    if (h.error) {
        const char* var = s->cfg.variant == ACG_VARIANT_INTERLEAVED ? "pcg_interleaved"
                                                                    : "pcg_standard";
        switch (h.error) {
            case kErrPivotFused:
                fail(ACG_ERR_BREAKDOWN,
                     "interleaved_prec_kernel: zero pivot in tridiagonal elimination");
            case kErrPivotPrecond:
                fail(ACG_ERR_BREAKDOWN, "precondition: zero pivot in tridiagonal elimination");
            case kErrPivotTridiag:
                fail(ACG_ERR_BREAKDOWN, "solve_tridiag_set: zero pivot in tridiagonal elimination");
            case kErrKappa:
                fail(ACG_ERR_BREAKDOWN, "%s: <r,z> not positive (preconditioner not SPD?)", var);
            default:
                fail(ACG_ERR_BREAKDOWN, "%s: <p,Ap> not positive (operator not SPD?)", var);
        }
    }
    // lagged catch-up u += alpha p when the interleaved loop converged (solver.hpp:345-351)
    if (s->cfg.variant == ACG_VARIANT_INTERLEAVED && h.converged && h.iterations >= 1) {
        s->timer.begin(kBlas);
        op_axpy<T>(c, T(0), &S, 0, false, s->p, s->u, false);
        s->timer.end(kBlas);
    }
    const double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - s->t0).count();
    // residual_norm of the backend (solver.hpp:119-121 / :138-140)
    T tr = s->csr ? op_true_residual_csr<T>(c, s->u, s->f, s->q) : op_true_residual<T>(c, s->u, s->f);
    if (u_out) op_copy<T>(c, s->u, u_out, nullptr);
    if (res) {
        std::memset(res, 0, sizeof(*res));
        res->iterations = h.iterations;
        res->converged = h.converged;
        res->true_residual = static_cast<double>(tr);
        res->n_residual = h.n_res;
        res->n_kappa = h.n_kap;
        res->n_alpha = h.n_alp;
        res->n_beta = h.n_bet;
        res->timings.total = total;
        res->timings.setup = s->setup_s;
        if (s->timer.on) {
            CK(cudaStreamSynchronize(c->stream));
            res->timings.spmv = s->timer.seconds(kSpmv);
            res->timings.prec = s->timer.seconds(kPrec);
            res->timings.blas = s->timer.seconds(kBlas);
            res->timings.fused_spmv = s->timer.seconds(kFusedSpmv);
            res->timings.fused_prec = s->timer.seconds(kFusedPrec);
        }
        res->kernel_launches = g_launches.load() - s->launches0;
    }
    const int counts[4] = {h.n_res, h.n_kap, h.n_alp, h.n_bet};
    drain_histories(s, counts);  // also orders the stream (true residual, u_out)
    double* outs[4] = {hr, hk, ha, hb};
    for (int a = 0; a < 4; ++a) {
        const size_t n = static_cast<size_t>(counts[a]);
        if (outs[a]) {
            if (n) std::memcpy(outs[a], s->hv[a].data(), n * sizeof(double));
        } else if (res) {  // library-owned copy, released by acg_solve_result_release
            double* d = static_cast<double*>(std::malloc(std::max<size_t>(n, 1) * sizeof(double)));
            if (!d) throw std::bad_alloc();
            if (n) std::memcpy(d, s->hv[a].data(), n * sizeof(double));
            res->history[a] = d;
        }
    }
}

}  // namespace

extern "C" {

acg_status acg_solver_create(acg_solver** out, const acg_context* c, const acg_solver_config* cfg) {
    return guarded([&] {
        check_ctx(c);
        if (!out) fail(ACG_ERR_INVALID_ARGUMENT, "null output");
        validate(cfg);
        DeviceGuard g(c->device);
        CtxLock lk(c);
        auto s = std::make_unique<acg_solver>();
        s->ctx = c;
        s->cfg = *cfg;
        ACG_TDISPATCH(c, solver_alloc<T>(s.get()));
        *out = s.release();
        c->user_solvers.push_back(*out);
    });
}

acg_status acg_solver_destroy(acg_solver* s) {
    return guarded([&] {
        if (!s) return;
        if (!s->ctx) {  // orphaned by acg_context_destroy: device resources already freed
            delete s;
            return;
        }
        const acg_context* c = s->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "solver of a destroyed context");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        auto& v = c->user_solvers;
        v.erase(std::remove(v.begin(), v.end(), s), v.end());
        cudaStreamSynchronize(c->stream);
        delete s;
    });
}

acg_status acg_solver_start(acg_solver* s, const acg_field* f, const acg_field* u0) {
    return guarded([&] {
        if (!s) fail(ACG_ERR_INVALID_ARGUMENT, "null solver");
        const acg_context* c = s->ctx;
        if (!c) fail(ACG_ERR_INVALID_ARGUMENT, "solver of a destroyed context");
        check_field(c, f, "solve");
        if (u0) check_field(c, u0, "solve");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        ACG_TDISPATCH(c, solver_start<T>(s, f, u0));
    });
}

acg_status acg_solver_iterate(acg_solver* s, int n) {
    return guarded([&] {
        if (!s || !s->started) fail(ACG_ERR_INVALID_ARGUMENT, "solver not started");
        if (!s->ctx) fail(ACG_ERR_INVALID_ARGUMENT, "solver of a destroyed context");
        DeviceGuard g(s->ctx->device);
        CtxLock lk(s->ctx);
        ACG_TDISPATCH(s->ctx, solver_iterate_drained<T>(s, n));
    });
}

acg_status acg_solver_time_kernels(acg_solver* s, int enable) {
    return guarded([&] {
        if (!s) fail(ACG_ERR_INVALID_ARGUMENT, "null solver");
        s->ktimer.on = enable != 0;
        s->ktimer.reset();
    });
}

acg_status acg_solver_kernel_times(acg_solver* s, int* n_prec, double* ms_prec, int* n_spmv,
                                   double* ms_spmv) {
    return guarded([&] {
        if (!s) fail(ACG_ERR_INVALID_ARGUMENT, "null solver");
        if (!s->ctx) fail(ACG_ERR_INVALID_ARGUMENT, "solver of a destroyed context");
        DeviceGuard g(s->ctx->device);
        CtxLock lk(s->ctx);
        CK(cudaStreamSynchronize(s->ctx->stream));
        if (n_prec) *n_prec = s->ktimer.count(kFusedPrec);
        if (ms_prec) *ms_prec = s->ktimer.seconds(kFusedPrec) * 1e3;
        if (n_spmv) *n_spmv = s->ktimer.count(kFusedSpmv);
        if (ms_spmv) *ms_spmv = s->ktimer.seconds(kFusedSpmv) * 1e3;
        s->ktimer.reset();
    });
}

acg_status acg_solver_finish(acg_solver* s, acg_field* u_out, acg_solve_result* res, double* hr,
                             double* hk, double* ha, double* hb) {
    return guarded([&] {
        if (!s || !s->started) fail(ACG_ERR_INVALID_ARGUMENT, "solver not started");
        if (!s->ctx) fail(ACG_ERR_INVALID_ARGUMENT, "solver of a destroyed context");
        if (u_out) check_field(s->ctx, u_out, "solve");
        DeviceGuard g(s->ctx->device);
        CtxLock lk(s->ctx);
        ACG_TDISPATCH(s->ctx, solver_finish<T>(s, u_out, res, hr, hk, ha, hb));
    });
}

acg_status acg_solve(const acg_context* c, const acg_field* f, const acg_field* u0,
                     const acg_solver_config* cfg, acg_field* u_out, acg_solve_result* res,
                     double* hr, double* hk, double* ha, double* hb) {
    return guarded([&] {
        check_ctx(c);
        check_field(c, f, "solve");
        if (u0) check_field(c, u0, "solve");
        if (u_out) check_field(c, u_out, "solve");
        validate(cfg);
        DeviceGuard g(c->device);
        CtxLock lk(c);
        ACG_TDISPATCH(c, {
            acg_solver* s = cached_solver<T>(c, cfg);
            solver_start<T>(s, f, u0);
            solver_run<T>(s);
            solver_finish<T>(s, u_out, res, hr, hk, ha, hb);
        });
    });
}

// ------------------------------------------------------- host entry points
acg_status acg_apply_host(const acg_context* c, acg_layout layout, const void* x, void* y) {
    return guarded([&] {
        check_ctx(c);
        if (!x || !y) fail(ACG_ERR_INVALID_ARGUMENT, "null buffer");
        if (x == y) fail(ACG_ERR_INVALID_ARGUMENT, "apply: x and y must not alias");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        PoolField fx(c), fy(c);
        ACG_TDISPATCH(c, {
            upload_t<T>(fx.f, x, layout, ACG_HOST_FULL);
            op_apply<T>(c, fx.f, fy.f, nullptr);
            download_t<T>(fy.f, y, layout, ACG_HOST_FULL);
        });
    });
}

acg_status acg_precondition_host(const acg_context* c, acg_layout layout, const void* y, void* x) {
    return guarded([&] {
        check_ctx(c);
        if (!x || !y) fail(ACG_ERR_INVALID_ARGUMENT, "null buffer");
        if (x == y) fail(ACG_ERR_INVALID_ARGUMENT, "precondition: y and x must not alias");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        PoolField fy(c), fx(c);
        ACG_TDISPATCH(c, {
            upload_t<T>(fy.f, y, layout, ACG_HOST_FULL);
            reset_tmp<T>(c);
            auto S = tmp_scalars<T>(c);
            op_precondition<T>(c, fy.f, fx.f, S, nullptr);
            CK(cudaPeekAtLastError());
            for (Scalars<T>* sp : S)
                if (read_scalars<T>(c, sp).pivot)
                    fail(ACG_ERR_BREAKDOWN, "precondition: zero pivot in tridiagonal elimination");
            download_t<T>(fx.f, x, layout, ACG_HOST_FULL);
        });
    });
}

acg_status acg_true_residual_host(const acg_context* c, acg_layout layout, const void* u,
                                  const void* f, double* out) {
    return guarded([&] {
        check_ctx(c);
        if (!u || !f || !out) fail(ACG_ERR_INVALID_ARGUMENT, "null buffer");
        DeviceGuard g(c->device);
        CtxLock lk(c);
        PoolField fu(c), ff(c);
        ACG_TDISPATCH(c, {
            upload_t<T>(fu.f, u, layout, ACG_HOST_FULL);
            upload_t<T>(ff.f, f, layout, ACG_HOST_FULL);
            *out = static_cast<double>(op_true_residual<T>(c, fu.f, ff.f));
        });
    });
}

acg_status acg_solve_host(const acg_context* c, acg_layout layout, const void* f, const void* u0,
                          const acg_solver_config* cfg, void* u_out, acg_solve_result* res,
                          double* hr, double* hk, double* ha, double* hb) {
    return guarded([&] {
        check_ctx(c);
        if (!f || !u_out) fail(ACG_ERR_INVALID_ARGUMENT, "null buffer");
        validate(cfg);
        DeviceGuard g(c->device);
        CtxLock lk(c);
        PoolField ff(c), fu0(c), fu(c);
        acg_solver_config cl = *cfg;
        cl.layout = layout;  // CsrBackend orders its rows by the fields' layout (solver.hpp:129)
        ACG_TDISPATCH(c, {
            upload_t<T>(ff.f, f, layout, ACG_HOST_FULL);
            if (u0) upload_t<T>(fu0.f, u0, layout, ACG_HOST_FULL);
            acg_solver* s = cached_solver<T>(c, &cl);
            solver_start<T>(s, ff.f, u0 ? fu0.f : nullptr);
            solver_run<T>(s);
            solver_finish<T>(s, fu.f, res, hr, hk, ha, hb);
            download_t<T>(fu.f, u_out, layout, ACG_HOST_FULL);
        });
    });
}

}  // extern "C"
