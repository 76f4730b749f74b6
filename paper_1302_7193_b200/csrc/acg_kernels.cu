// sm_100a kernels of the B200-native matrix-free PCG (arXiv 1302.7193).
//
//   K1 k_fused_prec     interleaved_prec_kernel   operator.hpp:272-346 (Alg. 3)
//   K2 k_fused_spmv     interleaved_spmv_kernel   operator.hpp:214-266 (Alg. 2)
//   K3 k_apply          apply                     operator.hpp:101-135
//   K4 k_precondition   precondition              operator.hpp:141-191
//   K5 k_axpy/k_scal/k_dot_partials  field.hpp:116-173
//   K6 k_tree1/k_tree2/k_finish      pairwise_sum parallel.hpp:11-20 + the
//                                    scalar recurrences of solver.hpp:288-364
//   K7 k_transpose      relayout / array_to_field field.hpp:102-109, bindings.cpp:40-59
//   K8 k_residual_partials  true_residual        solver.hpp:61-69 (one pass)
//   K11 k_fill_random   fill_random               field.hpp:180-196
//
// One thread owns one vertical column (paper Sec. 5, "one thread per column");
// a warp covers 32 consecutive j of one i-plane, so every level of every field
// is one coalesced row. Every arithmetic operation of the EXACT path is an
// explicit IEEE round-to-nearest intrinsic in the reference's association
// order (the reference builds with -ffp-contract=off), which makes the GPU
// bit-identical to the CPU. The FAST path allows FMA contraction and replaces
// the three divides per Thomas level by one reciprocal.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "acg_internal.h"

namespace acg {

std::atomic<long long> g_launches{0};

namespace {

// ------------------------------------------------------------- arithmetic
template <typename T, bool Fast>
struct Ar;
template <>
struct Ar<double, false> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};
template <>
struct Ar<float, false> {
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
};
template <typename T>
struct Ar<T, true> {
    static __device__ __forceinline__ T mul(T a, T b) { return a * b; }
    static __device__ __forceinline__ T add(T a, T b) { return a + b; }
    static __device__ __forceinline__ T sub(T a, T b) { return a - b; }
    static __device__ __forceinline__ T div(T a, T b) { return a / b; }
};

__device__ __forceinline__ double sqrt_rn(double x) { return __dsqrt_rn(x); }
__device__ __forceinline__ float sqrt_rn(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// Programmatic dependent launch: kernels launched with the PDL attribute may
// start while the previous kernel of the stream finishes; they must wait for it
// (griddepcontrol.wait, a no-op without the attribute) before reading its
// outputs. launch_dependents lets the next kernel's CTAs be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
// Reads of the device scalars a PDL kernel makes after pdl_wait(): the scalars
// are written by the immediately preceding kernel, so they must not come from
// a load the compiler hoisted above the wait (a const __restrict__ pointer is
// otherwise read through the non-coherent path, before griddepcontrol.wait).
template <typename V>
__device__ __forceinline__ V ld_dep(const V* p) {
    return *reinterpret_cast<const volatile V*>(p);
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Fused halo, consumer side: thread 0 acquires the neighbour's flag (set by its
// K1 after the boundary plane landed in this rank's mailbox), then the CTA
// proceeds. Traps after ~20 s instead of hanging when a peer never arrives.
__device__ __forceinline__ void halo_acquire(const unsigned long long* flag, unsigned long long seq) {
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        const long long t0 = clock64();
        while (ld_acquire_sys(flag) < seq) {
            if (clock64() - t0 > (40ll << 30)) __trap();
            __nanosleep(32);
        }
    }
    __syncthreads();
}

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("ACG_PDL");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline int grid_1d(long long n, int threads) {
    long long b = (n + threads - 1) / threads;
    const long long cap = 148LL * 32;
    return static_cast<int>(b < 1 ? 1 : (b > cap ? cap : b));
}

template <typename T>
__device__ __forceinline__ void load_profile(T* prof, const T* src, int count, int tid,
                                             int nthreads) {
    for (int t = tid; t < count; t += nthreads) prof[t] = src[t];
}

// 7-point stencil value (operator.hpp:127-132), summed left to right.
template <typename T, bool Fast>
__device__ __forceinline__ T stencil(T sA, T area, T adiag, T bk, T ck, T ae, T aw, T an, T as,
                                     T x0, T xu, T xd, T xe, T xw, T xn, T xs) {
    using A = Ar<T, Fast>;
    T t = A::mul(A::sub(A::mul(sA, area), adiag), x0);
    t = A::add(t, A::mul(A::mul(area, bk), xu));
    t = A::add(t, A::mul(A::mul(area, ck), xd));
    t = A::add(t, A::mul(ae, xe));
    t = A::add(t, A::mul(aw, xw));
    t = A::add(t, A::mul(an, xn));
    t = A::add(t, A::mul(as, xs));
    return t;
}

// Per-column stencil data (ColumnStencil, operator.hpp:75-94). Missing
// horizontal edges read the column's own value with a zero coefficient.
template <typename T>
struct Col {
    T area, adiag, ae, aw, an, as;
    long long oe, ow, on, os;
};

template <typename T>
__device__ __forceinline__ Col<T> load_col(const SlabView<T>& v, int il, int j) {
    const long long ncol = static_cast<long long>(v.m_loc) * v.m;
    const long long c = static_cast<long long>(il) * v.m + j;
    const int ig = v.i0 + il;
    Col<T> s;
    s.area = v.col[kColArea * ncol + c];
    s.adiag = v.col[kColDiag * ncol + c];
    s.ae = v.col[kColE * ncol + c];
    s.aw = v.col[kColW * ncol + c];
    s.an = v.col[kColN * ncol + c];
    s.as = v.col[kColS * ncol + c];
    s.oe = ig + 1 < v.m ? v.plane : 0;
    s.ow = ig > 0 ? -v.plane : 0;
    s.on = j + 1 < v.m ? 1 : 0;
    s.os = j > 0 ? -1 : 0;
    return s;
}

// Stage 1 of the reduction fused into a sweep's epilogue. When a CTA's NT
// columns are one aligned node of the reference's tree over the slab's column
// order (slab column count a power of two, CTA = NT consecutive columns of one
// i-plane), that node is a perfect binary tree over NT/8 sequential sums of 8
// (parallel.hpp:11-20: n <= 8 sequential, else split in halves). vals[a][col]
// holds the CTA's per-column partials in column order; warp 0 reduces them and
// writes stage[a * nleaves + leaf], exactly the value k_tree1 would produce
// for that node. Requires nv * NT / 8 <= 32.
template <typename T, int NT>
__device__ __forceinline__ void cta_subtree_sums(const T* vals, int nv, T* __restrict__ stage,
                                                 int nleaves, long long leaf) {
    constexpr int BT = NT / 8;                 // sequential blocks per array
    constexpr int L = BT > 32 ? BT / 32 : 1;   // blocks per lane (perfect tree in registers)
    constexpr int B = BT / L;                  // lanes per array
    static_assert(BT >= 1 && (BT & (BT - 1)) == 0 && L * B == BT, "power-of-two block count");
    const int lane = threadIdx.x;
    const int a = lane / B, b = lane % B;
    T v = T(0);
    if (a < nv) {
        T w[L];
#pragma unroll
        for (int i = 0; i < L; ++i) {
            const T* x = vals + a * NT + 8 * (b * L + i);
            w[i] = T(0);
#pragma unroll
            for (int l = 0; l < 8; ++l) w[i] = add_rn(w[i], x[l]);
        }
#pragma unroll
        for (int st = 1; st < L; st <<= 1)
#pragma unroll
            for (int i = 0; i + st < L; i += 2 * st) w[i] = add_rn(w[i], w[i + st]);
        v = w[0];
    }
#pragma unroll
    for (int w = 1; w < B; w <<= 1) {
        const T o = __shfl_down_sync(0xffffffffu, v, w, B);
        if (b % (2 * w) == 0) v = add_rn(v, o);
    }
    if (a < nv && b == 0) stage[a * static_cast<long long>(nleaves) + leaf] = v;
}

template <typename T>
__device__ void run_op(Scalars<T>* S, int op, const T* sums, bool push = true);

// Consumed-reduction prologue (Consume, acg_internal.h): the whole CTA reduces
// the previous sweep's nleaves tree leaves — c consecutive leaves per thread,
// a shuffle tree per warp, a tree over the warps: the perfect tree
// k_tree2_wide evaluates, so the same bits — while its last warp fetches the
// state cs.in into shared memory, one word per thread; thread 0 runs the
// scalar program there and CTA (0, 0) stores the result to cs.out. `red`: 64
// values of shared memory the CTA does not use yet.
template <typename T>
struct Consumed {
    T alpha, beta;
    int done;
};

template <typename T, int NT>
__device__ Consumed<T> consume_finish(const Consume<T>& cs, int tid, T* red) {
    constexpr int CM = kConsumeMaxLeaves / NT;  // most leaves per thread
    constexpr int NW = static_cast<int>(sizeof(Scalars<T>) / 8);
    static_assert(CM >= 1 && NT % 32 == 0 && NW <= 32, "consume_finish: CTA shape");
    static_assert(sizeof(Scalars<T>) % 8 == 0, "Scalars: whole 8-byte words");
    __shared__ Consumed<T> res;
    __shared__ __align__(8) unsigned long long state[NW];
    // the last warp also fetches the state words, one each, while the leaves load
    if (tid >= NT - 32 && tid - (NT - 32) < NW)
        state[tid - (NT - 32)] =
            __ldcg(reinterpret_cast<const unsigned long long*>(cs.in) + (tid - (NT - 32)));
    const int nl = cs.nleaves;
    const int c = nl > NT ? nl / NT : 1;
    const int nt = nl / c;  // threads holding leaves (power of two)
    const int lane = tid & 31, warp = tid >> 5;
    const int width = nt < 32 ? nt : 32;
    for (int a = 0; a < cs.nv; ++a) {
        T v[CM];
        const T* lf = cs.leaves + static_cast<long long>(a) * nl + tid * c;
#pragma unroll
        for (int l = 0; l < CM; ++l) v[l] = (tid < nt && l < c) ? __ldcg(lf + l) : T(0);
#pragma unroll
        for (int w = 1; w < CM; w <<= 1)
#pragma unroll
            for (int l = 0; l + w < CM; l += 2 * w)
                if (w < c) v[l] = add_rn(v[l], v[l + w]);
        T x = v[0];
        for (int w = 1; w < width; w <<= 1) {
            const T o = __shfl_down_sync(0xffffffffu, x, w, width);
            if ((lane & (2 * w - 1)) == 0) x = add_rn(x, o);
        }
        if (lane == 0 && tid < nt) red[a * 32 + warp] = x;
    }
    __syncthreads();
    if (tid == 0) {
        T sums[4] = {T(0), T(0), T(0), T(0)};
        const int nw = (nt + 31) / 32;
        for (int a = 0; a < cs.nv; ++a) {
            for (int st = 1; st < nw; st <<= 1)
                for (int w = 0; w + st < nw; w += 2 * st)
                    red[a * 32 + w] = add_rn(red[a * 32 + w], red[a * 32 + w + st]);
            sums[a] = red[a * 32];
        }
        Scalars<T>* loc = reinterpret_cast<Scalars<T>*>(state);  // the program runs in shared memory
        const bool lead = blockIdx.x == 0 && blockIdx.y == 0;
        if (loc->pend && !loc->done) run_op(loc, cs.op, sums, lead);
        res.alpha = loc->alpha;
        res.beta = loc->beta;
        res.done = loc->done;
        loc->pend = loc->done ? 0 : 1;  // this sweep's leaves follow unless it is skipped
    }
    __syncthreads();
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid < NW)  // CTA (0, 0): the next state
        reinterpret_cast<unsigned long long*>(cs.out)[tid] = state[tid];
    return res;
}

// ================================================================ K1 / K4
#include "acg_thomas.cuh"
#include "acg_thomas_tm.cuh"
#include "acg_thomas_tm2.cuh"

// ================================================================ K2 / K3 / K8
constexpr int kStencilWarps = 8;

// K3: y = A x (operator.hpp:124-133)
template <typename T, bool Fast>
__global__ void __launch_bounds__(32 * kStencilWarps)
    k_apply(const SlabView<T> v, const T* __restrict__ x, T* __restrict__ y,
            const Scalars<T>* __restrict__ gate) {
    using A = Ar<T, Fast>;
    if (gate && gate->done) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* prof = reinterpret_cast<T*>(smem_raw);
    const int n_z = v.n_z, m = v.m;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    load_profile(prof, v.prof, 4 * n_z, tid, 32 * kStencilWarps);
    __syncthreads();
    const int j = blockIdx.x * 32 + threadIdx.x;
    const int il = blockIdx.y * kStencilWarps + threadIdx.y;
    if (j >= m || il >= v.m_loc) return;
    const T* sP = prof + kProfS * n_z;
    const T* bP = prof + kProfB * n_z;
    const T* cP = prof + kProfC * n_z;
    const T* dP = prof + kProfD * n_z;
    const Col<T> c = load_col(v, il, j);
    const long long base = static_cast<long long>(il) * v.plane + j;
    const T* xc = x + base;
    T* yc = y + base;
    T x0 = xc[0], xd = x0;
#pragma unroll 4
    for (int k = 0; k < n_z; ++k) {
        const long long l = static_cast<long long>(k) * m;
        const T xu = (k + 1 < n_z) ? xc[l + m] : x0;
        const T t = stencil<T, Fast>(sP[k], c.area, c.adiag, bP[k], cP[k], c.ae, c.aw, c.an, c.as,
                                     x0, xu, xd, xc[l + c.oe], xc[l + c.ow], xc[l + c.on],
                                     xc[l + c.os]);
        __stcs(yc + l, A::mul(t, dP[k]));
        xd = x0;
        x0 = xu;
    }
}

// K8: per-column sum of (f - A u)^2 — true_residual (solver.hpp:61-69) in one
// pass: -t is exact and f + (-t) == f - t, so this equals apply+scal+axpy+nrm2.
template <typename T, bool Fast>
__global__ void __launch_bounds__(32 * kStencilWarps)
    k_residual_partials(const SlabView<T> v, const T* __restrict__ u, const T* __restrict__ f,
                        T* __restrict__ part) {
    using A = Ar<T, Fast>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* prof = reinterpret_cast<T*>(smem_raw);
    const int n_z = v.n_z, m = v.m;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    load_profile(prof, v.prof, 4 * n_z, tid, 32 * kStencilWarps);
    __syncthreads();
    const int j = blockIdx.x * 32 + threadIdx.x;
    const int il = blockIdx.y * kStencilWarps + threadIdx.y;
    if (j >= m || il >= v.m_loc) return;
    const T* sP = prof + kProfS * n_z;
    const T* bP = prof + kProfB * n_z;
    const T* cP = prof + kProfC * n_z;
    const T* dP = prof + kProfD * n_z;
    const Col<T> c = load_col(v, il, j);
    const long long base = static_cast<long long>(il) * v.plane + j;
    const T* uc = u + base;
    const T* fc = f + base;
    T x0 = uc[0], xd = x0, sum = T(0);
#pragma unroll 4
    for (int k = 0; k < n_z; ++k) {
        const long long l = static_cast<long long>(k) * m;
        const T xu = (k + 1 < n_z) ? uc[l + m] : x0;
        const T t = A::mul(stencil<T, Fast>(sP[k], c.area, c.adiag, bP[k], cP[k], c.ae, c.aw, c.an,
                                            c.as, x0, xu, xd, uc[l + c.oe], uc[l + c.ow],
                                            uc[l + c.on], uc[l + c.os]),
                           dP[k]);
        const T r = A::sub(__ldcs(fc + l), t);
        sum = A::add(sum, A::mul(r, r));
        xd = x0;
        x0 = xu;
    }
    part[static_cast<long long>(il) * m + j] = sum;
}

// per-column dot partials in ascending k (field.hpp:134-153)
template <typename T>
__global__ void __launch_bounds__(256)
    k_dot_partials(const SlabView<T> v, const T* __restrict__ x, const T* __restrict__ y,
                   T* __restrict__ part, const Scalars<T>* __restrict__ gate) {
    using A = Ar<T, false>;
    if (gate && gate->done) return;
    const int j = blockIdx.x * 32 + threadIdx.x;
    const int il = blockIdx.y * 8 + threadIdx.y;
    if (j >= v.m || il >= v.m_loc) return;
    const long long base = static_cast<long long>(il) * v.plane + j;
    T s = T(0);
#pragma unroll 4
    for (int k = 0; k < v.n_z; ++k) {
        const long long l = base + static_cast<long long>(k) * v.m;
        s = A::add(s, A::mul(__ldcs(x + l), __ldcs(y + l)));
    }
    part[static_cast<long long>(il) * v.m + j] = s;
}

// ================================================================ K5 BLAS-1
template <typename T>
__global__ void k_axpy(long long n, T value, const T* __restrict__ coef, int neg,
                       const T* __restrict__ x, T* __restrict__ y,
                       const Scalars<T>* __restrict__ gate) {
    using A = Ar<T, false>;
    if (gate && gate->done) return;
    T a = coef ? *coef : value;
    if (neg) a = -a;
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < n;
         l += (long long)gridDim.x * blockDim.x)
        y[l] = A::add(A::mul(a, x[l]), y[l]);
}

template <typename T>
__global__ void k_scal(long long n, T value, const T* __restrict__ coef, T* __restrict__ x,
                       const Scalars<T>* __restrict__ gate) {
    using A = Ar<T, false>;
    if (gate && gate->done) return;
    const T a = coef ? *coef : value;
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < n;
         l += (long long)gridDim.x * blockDim.x)
        x[l] = A::mul(a, x[l]);
}

template <typename T>
__global__ void k_copy(long long n, const T* __restrict__ x, T* __restrict__ y,
                       const Scalars<T>* __restrict__ gate) {
    if (gate && gate->done) return;
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < n;
         l += (long long)gridDim.x * blockDim.x)
        y[l] = x[l];
}

template <typename T>
__global__ void k_fill(long long n, T value, T* __restrict__ x) {
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < n;
         l += (long long)gridDim.x * blockDim.x)
        x[l] = value;
}

// K11: draw number n = (i*m + j)*n_z + k of the sequential splitmix64 stream
// (field.hpp:180-196): state_n = seed + (n+1)*golden, so every element is
// generated independently and the field matches the host fill bit for bit.
template <typename T>
__global__ void k_fill_random(const SlabView<T> v, uint64_t seed, T* __restrict__ x) {
    const long long total = static_cast<long long>(v.m_loc) * v.plane;
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < total;
         l += (long long)gridDim.x * blockDim.x) {
        const long long il = l / v.plane;
        const long long rem = l - il * v.plane;
        const long long k = rem / v.m;
        const long long j = rem - k * v.m;
        const unsigned long long nidx =
            (static_cast<unsigned long long>(v.i0 + il) * v.m + j) * v.n_z + k;
        unsigned long long s = seed + (nidx + 1ull) * 0x9e3779b97f4a7c15ull;
        s = (s ^ (s >> 30)) * 0xbf58476d1ce4e5b9ull;
        s = (s ^ (s >> 27)) * 0x94d049bb133111ebull;
        s = s ^ (s >> 31);
        const double u = __dmul_rn(static_cast<double>(s >> 11), 0x1.0p-53);
        x[l] = static_cast<T>(__dsub_rn(__dmul_rn(2.0, u), 1.0));
    }
}

// ================================================================ K7 relayout
template <typename T>
__global__ void k_transpose(const T* __restrict__ in, T* __restrict__ out, int nx, int ny, int nb,
                            long long isy, long long isb, long long osx, long long osb) {
    __shared__ T tile[32][33];
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    for (int b = blockIdx.z; b < nb; b += gridDim.z) {
        for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
            const int x = x0 + threadIdx.x, y = y0 + dy;
            if (x < nx && y < ny) tile[dy][threadIdx.x] = in[x + y * isy + b * isb];
        }
        __syncthreads();
        for (int dx = threadIdx.y; dx < 32; dx += blockDim.y) {
            const int y = y0 + threadIdx.x, x = x0 + dx;
            if (x < nx && y < ny) out[x * osx + y + b * osb] = tile[threadIdx.x][dx];
        }
        __syncthreads();
    }
}

// ================================================================ K6 reductions
__device__ __forceinline__ void node_range(long long n, int depth, long long t, long long& lo,
                                           long long& hi) {
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

// pairwise_sum of a node of size <= 16 (parallel.hpp:11-20)
template <typename T>
__device__ __forceinline__ T leaf_sum(const T* v, long long n) {
    auto seq = [](const T* a, long long c) {
        T s = T(0);
        for (long long l = 0; l < c; ++l) s = add_rn(s, a[l]);
        return s;
    };
    if (n <= 8) return seq(v, n);
    const long long h = n / 2;
    return add_rn(seq(v, h), seq(v + h, n - h));
}

template <typename T>
__global__ void __launch_bounds__(256)
    k_tree1(long long n, int depth, const T* __restrict__ in0, const T* __restrict__ in1,
            const T* __restrict__ in2, int nv, T* __restrict__ stage, int nblocks,
            const Scalars<T>* __restrict__ gate) {
    if (gate && gate->done) return;
    __shared__ T sh[3][256];
    const int tid = threadIdx.x;
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + tid;
    long long lo, hi;
    node_range(n, depth, t, lo, hi);
    const T* ins[3] = {in0, in1, in2};
    for (int a = 0; a < nv; ++a) sh[a][tid] = leaf_sum(ins[a] + lo, hi - lo);
    __syncthreads();
    for (int s = 1; s < static_cast<int>(blockDim.x); s <<= 1) {
        if ((tid & (2 * s - 1)) == 0)
            for (int a = 0; a < nv; ++a) sh[a][tid] = add_rn(sh[a][tid], sh[a][tid + s]);
        __syncthreads();
    }
    if (tid == 0)
        for (int a = 0; a < nv; ++a) stage[a * nblocks + blockIdx.x] = sh[a][0];
}

// Scalar recurrences of the PCG drivers (solver.hpp:288-364); every value
// is computed in T and pushed to the histories as double, as in the reference.
// One history entry: the count always advances, the store only where `push`
// (consumed-reduction mode: every CTA runs the program, CTA (0, 0) records).
__device__ __forceinline__ void hist(double* h, int& n, int mask, double x, bool push) {
    if (push) h[n & mask] = x;
    ++n;
}

template <typename T>
__device__ void run_op(Scalars<T>* S, int op, const T* sums, bool push) {
    using A = Ar<T, false>;
    S->pend = 0;
    switch (op) {
        case kOpStore:
            for (int a = 0; a < 4; ++a) S->val[a] = sums[a];
            break;
        case kOpR0: {
            const T rn = sqrt_rn(sums[0]);
            S->r_norm = rn;
            S->r0 = rn;
            hist(S->h_res, S->n_res, S->hmask, static_cast<double>(rn), push);
            if (static_cast<double>(rn) <= S->tau) {
                S->converged = 1;
                S->done = 1;
            }
        } break;
        case kOpKappa0: {
            if (S->pivot) {
                S->error = S->pivot == 2 ? kErrPivotTridiag : kErrPivotPrecond;
                S->done = 1;
                break;
            }
            S->kappa_old = sums[0];
            hist(S->h_kap, S->n_kap, S->hmask, static_cast<double>(sums[0]), push);
            if (!(static_cast<double>(sums[0]) > 0.0)) {
                S->error = kErrKappa;
                S->done = 1;
            }
        } break;
        case kOpSigma0:
        case kOpIlSpmv:
        case kOpStdSigma: {
            S->sigma = sums[0];
            if (!(static_cast<double>(sums[0]) > 0.0)) {
                S->error = kErrSigma;
                S->done = 1;
                break;
            }
            const T al = A::div(S->kappa_old, sums[0]);
            S->alpha = al;
            S->neg_alpha = -al;
            hist(S->h_alp, S->n_alp, S->hmask, static_cast<double>(al), push);
            if (op == kOpSigma0) {
                S->it = 1;
            } else if (op == kOpIlSpmv) {
                if (++S->it > S->maxiter) S->done = 1;
            }
        } break;
        case kOpIlPrec: {
            if (S->pivot) {
                S->error = kErrPivotFused;
                S->done = 1;
                break;
            }
            const T rn = sqrt_rn(sums[0]);
            const T ka = sums[1];
            S->r_norm = rn;
            S->kappa = ka;
            hist(S->h_res, S->n_res, S->hmask, static_cast<double>(rn), push);
            S->iterations = S->it;
            if (static_cast<double>(rn) / static_cast<double>(S->r0) < S->eps ||
                static_cast<double>(rn) < S->tau) {
                S->converged = 1;
                S->done = 1;
                break;
            }
            hist(S->h_kap, S->n_kap, S->hmask, static_cast<double>(ka), push);
            const T be = A::div(ka, S->kappa_old);
            S->beta = be;
            hist(S->h_bet, S->n_bet, S->hmask, static_cast<double>(be), push);
            S->kappa_old = ka;
        } break;
        case kOpStdRnorm: {
            const T rn = sqrt_rn(sums[0]);
            S->r_norm = rn;
            hist(S->h_res, S->n_res, S->hmask, static_cast<double>(rn), push);
            S->iterations = S->it;
            if (static_cast<double>(rn) / static_cast<double>(S->r0) < S->eps ||
                static_cast<double>(rn) < S->tau) {
                S->converged = 1;
                S->done = 1;
            }
        } break;
        case kOpStdKappa: {
            if (S->pivot) {
                S->error = S->pivot == 2 ? kErrPivotTridiag : kErrPivotPrecond;
                S->done = 1;
                break;
            }
            const T ka = sums[0];
            S->kappa = ka;
            hist(S->h_kap, S->n_kap, S->hmask, static_cast<double>(ka), push);
            const T be = A::div(ka, S->kappa_old);
            S->beta = be;
            hist(S->h_bet, S->n_bet, S->hmask, static_cast<double>(be), push);
            S->kappa_old = ka;
            if (++S->it > S->maxiter) S->done = 1;
        } break;
        default:
            break;
    }
}

// Combine the slab sums of one value: the perfect tree above the slab nodes
// when the slabs are nodes of the reference tree, else the pairwise rule.
template <typename T>
__device__ T combine_slabs(const T* gather, int a, int nslabs, bool exact) {
    if (nslabs == 1) return gather[a];
    T v[64];
    for (int s = 0; s < nslabs; ++s) v[s] = gather[s * 4 + a];
    if (exact) {
        for (int w = 1; w < nslabs; w <<= 1)
            for (int s = 0; s + w < nslabs; s += 2 * w) v[s] = add_rn(v[s], v[s + w]);
        return v[0];
    }
    // iterative pairwise_sum over nslabs values (explicit stack)
    long long st_lo[16], st_n[16];
    T st_acc[16];
    int st_state[16];
    int sp = 0;
    st_lo[0] = 0;
    st_n[0] = nslabs;
    st_state[0] = 0;
    T ret = T(0);
    while (sp >= 0) {
        const long long lo = st_lo[sp], n = st_n[sp];
        if (n <= 8) {
            T s = T(0);
            for (long long l = 0; l < n; ++l) s = add_rn(s, v[lo + l]);
            ret = s;
            --sp;
            continue;
        }
        if (st_state[sp] == 0) {
            st_state[sp] = 1;
            ++sp;
            st_lo[sp] = lo;
            st_n[sp] = n / 2;
            st_state[sp] = 0;
        } else if (st_state[sp] == 1) {
            st_acc[sp] = ret;
            st_state[sp] = 2;
            ++sp;
            st_lo[sp] = lo + n / 2;
            st_n[sp] = n - n / 2;
            st_state[sp] = 0;
        } else {
            ret = add_rn(st_acc[sp], ret);
            --sp;
        }
    }
    return ret;
}

template <typename T>
__global__ void __launch_bounds__(1024)
    k_tree2(int nleaves, const T* __restrict__ stage, int nv, T* __restrict__ gather, int slab,
            int finish, int nslabs, int exact, Scalars<T>* __restrict__ S, int op) {
    if (op != kOpStore && S->done) return;
    __shared__ T sh[3][1024];
    const int tid = threadIdx.x;
    const int nt = blockDim.x;
    const int c = nleaves / nt;  // leaves per thread, power of two <= 16
    for (int a = 0; a < nv; ++a) {
        T v[16];
        for (int l = 0; l < c; ++l) v[l] = stage[a * nleaves + tid * c + l];
        for (int w = 1; w < c; w <<= 1)
            for (int l = 0; l + w < c; l += 2 * w) v[l] = add_rn(v[l], v[l + w]);
        sh[a][tid] = v[0];
    }
    __syncthreads();
    for (int s = 1; s < nt; s <<= 1) {
        if ((tid & (2 * s - 1)) == 0)
            for (int a = 0; a < nv; ++a) sh[a][tid] = add_rn(sh[a][tid], sh[a][tid + s]);
        __syncthreads();
    }
    if (tid == 0) {
        for (int a = 0; a < nv; ++a) gather[slab * 4 + a] = sh[a][0];
        if (finish) {
            T sums[4] = {T(0), T(0), T(0), T(0)};
            for (int a = 0; a < nv; ++a) sums[a] = combine_slabs(gather, a, nslabs, exact != 0);
            run_op(S, op, sums);
        }
    }
}

// Stage 2 with warp shuffles: NTH threads, C consecutive leaves each (perfect
// tree in registers), then a shuffle tree per warp and a perfect tree over the
// warps — the same perfect tree over nleaves = NTH * C leaves as k_tree2.

template <typename T, int C>
__global__ void __launch_bounds__(256)
    k_tree2_shfl(int nleaves, const T* __restrict__ stage, int nv, T* __restrict__ gather,
                 int slab, int finish, int nslabs, int exact, Scalars<T>* __restrict__ S, int op,
                 const IpcPut<T> put) {
    pdl_trigger();  // the next sweep may start its prologue while this tree runs
    pdl_wait();
    // peer-memory ranks: the slab sums go straight into every rank's mailbox
    // (put.n > 0). The put is unconditional (a finished solve still keeps the
    // ranks' flag sequence in step), the reduction itself is gated.
    if (op != kOpStore && S->done) {
        if (put.n > 0 && threadIdx.x == 0) {
            __threadfence_system();
            for (int q = 0; q < put.n; ++q) st_release_sys(put.flag[q] + put.rank, put.seq);
        }
        return;
    }
    __shared__ T wsum[3][8];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int width = nt < 32 ? nt : 32;
    for (int a = 0; a < nv; ++a) {
        T v[C];
#pragma unroll
        for (int l = 0; l < C; ++l) v[l] = stage[a * static_cast<long long>(nleaves) + tid * C + l];
#pragma unroll
        for (int w = 1; w < C; w <<= 1)
#pragma unroll
            for (int l = 0; l + w < C; l += 2 * w) v[l] = add_rn(v[l], v[l + w]);
        T x = v[0];
        for (int w = 1; w < width; w <<= 1) {
            const T o = __shfl_down_sync(0xffffffffu >> (32 - width), x, w, width);
            if ((lane & (2 * w - 1)) == 0) x = add_rn(x, o);
        }
        if (lane == 0) wsum[a][warp] = x;
    }
    __syncthreads();
    if (tid == 0) {
        const int nw = (nt + 31) / 32;
        T sums[4] = {T(0), T(0), T(0), T(0)};
        for (int a = 0; a < nv; ++a) {
            T w8[8];
            for (int w = 0; w < nw; ++w) w8[w] = wsum[a][w];
            for (int st = 1; st < nw; st <<= 1)
                for (int w = 0; w + st < nw; w += 2 * st) w8[w] = add_rn(w8[w], w8[w + st]);
            gather[slab * 4 + a] = w8[0];
        }
        if (finish) {
            for (int a = 0; a < nv; ++a) sums[a] = combine_slabs(gather, a, nslabs, exact != 0);
            run_op(S, op, sums);
        }
    }
    if (put.n > 0 && tid == 0) {  // rank `put.rank`'s 4 sums into every mailbox, then the flags
        for (int q = 0; q < put.n; ++q) {
            T* d = put.dst[q] + put.rank * 4;
            for (int a = 0; a < 4; ++a) d[a] = gather[slab * 4 + a];
        }
        __threadfence_system();
        for (int q = 0; q < put.n; ++q) st_release_sys(put.flag[q] + put.rank, put.seq);
    }
}

// Peer-memory ranks: acquire flags[q] >= seq for every rank q (traps after
// ~20 s instead of hanging when a peer never arrives).
__device__ __forceinline__ void ipc_wait_all(const unsigned long long* flags, int n,
                                             unsigned long long seq) {
    const long long t0 = clock64();
    for (int q = 0; q < n; ++q)
        while (ld_acquire_sys(flags + q) < seq) {
            if (clock64() - t0 > (40ll << 30)) __trap();
            __nanosleep(32);
        }
    __threadfence_system();
}

// Perfect tree over blockDim.x * C consecutive leaves of nv (<= 2) arrays
// (array a at src + a * stride): C leaves per thread with 16-byte loads, the
// register tree, a shuffle tree per warp and a shuffle tree over the
// (power-of-two many) warps — the reference's pairwise tree restricted to an
// aligned perfect subtree. Lane 0 of warp 0 returns the sums in out[].
template <typename T, int C>
__device__ __forceinline__ void block_tree(const T* __restrict__ src, long long stride, int nv,
                                           T (&out)[2]) {
    __shared__ T wsum[2][32];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int width = nt < 32 ? nt : 32;
    T v[2][C];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        if (a < nv) {
            const T* p = src + a * stride + tid * C;
            if constexpr (C % 2 == 0 && sizeof(T) == 8) {
#pragma unroll
                for (int l = 0; l < C; l += 2) {
                    const double2 d = __ldcg(reinterpret_cast<const double2*>(p + l));
                    v[a][l] = d.x;
                    v[a][l + 1] = d.y;
                }
            } else {
#pragma unroll
                for (int l = 0; l < C; ++l) v[a][l] = __ldcg(p + l);
            }
        }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        if (a < nv) {
#pragma unroll
            for (int w = 1; w < C; w <<= 1)
#pragma unroll
                for (int l = 0; l + w < C; l += 2 * w) v[a][l] = add_rn(v[a][l], v[a][l + w]);
            T x = v[a][0];
            for (int w = 1; w < width; w <<= 1) {
                const T o = __shfl_down_sync(0xffffffffu >> (32 - width), x, w, width);
                if ((lane & (2 * w - 1)) == 0) x = add_rn(x, o);
            }
            if (lane == 0) wsum[a][warp] = x;
        }
    }
    const int nw = (nt + 31) / 32;  // a power of two
    __syncthreads();
    if (warp == 0) {
        for (int a = 0; a < nv; ++a) {
            T x = lane < nw ? wsum[a][lane] : T(0);
            for (int w = 1; w < nw; w <<= 1) {
                const T o = __shfl_down_sync(0xffffffffu, x, w);
                if ((lane & (2 * w - 1)) == 0) x = add_rn(x, o);
            }
            out[a] = x;
        }
    }
}

// Stage 1.5 for more than 8192 leaves: CTA b reduces leaves [b * 8192, (b+1) * 8192)
// (an aligned node of the tree) to mid[a * gridDim.x + b].
template <typename T>
__global__ void __launch_bounds__(1024)
    k_tree_mid(int nleaves, const T* __restrict__ stage, int nv, T* __restrict__ mid) {
    pdl_trigger();
    pdl_wait();
    T out[2];
    block_tree<T, 8>(stage + static_cast<long long>(blockIdx.x) * 8192, nleaves, nv, out);
    if (threadIdx.x == 0)
        for (int a = 0; a < nv; ++a) mid[a * gridDim.x + blockIdx.x] = out[a];
}

// Stage 2, wide (nv <= 2): up to 1024 threads with C (<= 8) consecutive
// leaves each (block_tree), then the finish / peer-memory put.
template <typename T, int C>
__global__ void __launch_bounds__(1024)
    k_tree2_wide(int nleaves, const T* __restrict__ stage, int nv, T* __restrict__ gather,
                 int slab, int finish, int nslabs, int exact, Scalars<T>* __restrict__ S, int op,
                 const IpcPut<T> put) {
    pdl_trigger();  // the next sweep may start its prologue while this tree runs
    pdl_wait();
    if (op != kOpStore && S->done) {  // gated; the peer-memory flags stay in lockstep
        if (put.n > 0 && threadIdx.x == 0) {
            __threadfence_system();
            for (int q = 0; q < put.n; ++q) st_release_sys(put.flag[q] + put.rank, put.seq);
            // still wait for every rank: no rank may run two reductions ahead and
            // overwrite a mailbox parity a peer is still reading
            if (put.wait != nullptr) ipc_wait_all(put.wait, put.n, put.seq);
        }
        return;
    }
    T out[2];
    block_tree<T, C>(stage, nleaves, nv, out);
    if (threadIdx.x == 0) {
        for (int a = 0; a < nv; ++a) gather[slab * 4 + a] = out[a];
        if (finish) {
            T sums[4] = {T(0), T(0), T(0), T(0)};
            for (int a = 0; a < nv; ++a) sums[a] = combine_slabs(gather, a, nslabs, exact != 0);
            run_op(S, op, sums);
        }
        if (put.n > 0) {  // rank `put.rank`'s 4 sums into every mailbox, then the flags
            for (int q = 0; q < put.n; ++q) {
                T* d = put.dst[q] + put.rank * 4;
                for (int a = 0; a < 4; ++a) d[a] = gather[slab * 4 + a];
            }
            __threadfence_system();
            for (int q = 0; q < put.n; ++q) st_release_sys(put.flag[q] + put.rank, put.seq);
            if (put.wait != nullptr) {  // every rank's sums have landed: finish here
                ipc_wait_all(put.wait, put.n, put.seq);
                T sums[4] = {T(0), T(0), T(0), T(0)};
                for (int a = 0; a < nv; ++a) sums[a] = combine_slabs(put.all, a, put.n, exact != 0);
                run_op(S, op, sums);
            }
        }
    }
}

template <typename T>
__global__ void k_finish(const T* __restrict__ gather, int nv, int nslabs, int exact,
                         Scalars<T>* __restrict__ S, int op, const unsigned long long* wait_flags,
                         unsigned long long seq) {
    if (wait_flags) {  // peer-memory ranks: every rank's sums have landed in this mailbox
        const long long t0 = clock64();
        for (int q = 0; q < nslabs; ++q)
            while (ld_acquire_sys(wait_flags + q) < seq) {
                if (clock64() - t0 > (40ll << 30)) __trap();
                __nanosleep(32);
            }
        __threadfence_system();
    }
    if (op != kOpStore && S->done) return;
    T sums[4] = {T(0), T(0), T(0), T(0)};
    for (int a = 0; a < nv; ++a) sums[a] = combine_slabs(gather, a, nslabs, exact != 0);
    run_op(S, op, sums);
}

// ------------------------------------------------------- peer-memory transport

struct FlagPtrs {
    unsigned long long* f[8];
};

__global__ void k_ipc_signal(FlagPtrs fp, int n, unsigned long long seq) {
    __threadfence_system();  // the data this flag publishes (copies earlier on the stream)
    for (int i = 0; i < n; ++i)
        if (fp.f[i]) st_release_sys(fp.f[i], seq);
}

__global__ void k_ipc_wait(const unsigned long long* flags, int n, unsigned long long need,
                           unsigned long long seq) {
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (!((need >> i) & 1ull)) continue;
        while (ld_acquire_sys(flags + i) < seq) {
            if (clock64() - t0 > (40ll << 30)) __trap();  // a peer never arrived: fail, do not hang
            __nanosleep(64);
        }
    }
    __threadfence_system();
}


// --------------------------------------------------------- launch helpers
inline void post_launch(const char* what) {
    ++g_launches;
    const cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) {
        std::fprintf(stderr, "acg: launch of %s failed: %s\n", what, cudaGetErrorString(e));
    }
}

#include "acg_stencil_tile.cuh"

// Opt a kernel in to more than 48 KB of dynamic shared memory. The attribute is
// set once per kernel and size (a driver call per launch costs host time the
// small grids, which are host-paced, cannot afford).
template <typename KernelT>
void ensure_smem(KernelT kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return;
    struct Applied {
        const void* kernel;
        int device;
        size_t bytes;
    };
    static std::mutex mu;
    static std::vector<Applied> set;  // attributes are per device context
    const void* key = reinterpret_cast<const void*>(kernel);
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    for (Applied& e : set)
        if (e.kernel == key && e.device == dev) {
            if (e.bytes >= bytes) return;
            e.bytes = bytes;
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes));
            return;
        }
    set.push_back({key, dev, bytes});
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(bytes));
}


// Thomas launch configuration of the global-memory fallback k_thomas (warps per
// block, phi checkpoint stride, cp.async depth), per precision.
using ThomasF64 = ThomasCfg<4, 4, 7>;
using ThomasF32 = ThomasCfg<4, 2, 7>;
template <typename T>
struct ThomasOf;
template <>
struct ThomasOf<double> { using type = ThomasF64; };
template <>
struct ThomasOf<float> { using type = ThomasF32; };

template <typename T, bool Fast, bool Fused, class C>
void launch_thomas_cfg(const SlabView<T>& v, T* r, const T* in, T* out, T* p2, T* pk,
                       Scalars<T>* S, const Scalars<T>* gate, T* phi_scratch, cudaStream_t st) {
    const dim3 block(32, C::W);
    const dim3 grid((v.m + 31) / 32, (v.m_loc + C::W - 1) / C::W);
    const size_t smem = thomas_smem_bytes<T, C>(v.n_z, phi_scratch != nullptr);
    if (phi_scratch) {
        ensure_smem(k_thomas<T, Fast, Fused, C, true>, smem);
        k_thomas<T, Fast, Fused, C, true>
            <<<grid, block, smem, st>>>(v, r, in, out, p2, pk, S, gate, phi_scratch);
    } else {
        ensure_smem(k_thomas<T, Fast, Fused, C, false>, smem);
        k_thomas<T, Fast, Fused, C, false>
            <<<grid, block, smem, st>>>(v, r, in, out, p2, pk, S, gate, phi_scratch);
    }
}

// Leaves of the reduction tree a sweep can emit directly (cta_subtree_sums):
// CTAs of `cols` consecutive columns of one i-plane, slab column count a power
// of two (so every CTA is an aligned node), at most kMaxFusedLeaves leaves
// (k_tree2_wide; above 8192 via the k_tree_mid nodes).
// 0: the sweep writes per-column partials and k_tree1 runs instead.
inline int num_sms() {
    static int n = [] {
        int dev = 0, c = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
        return c;
    }();
    return n;
}

template <typename T>
int fused_leaves(const SlabView<T>& v, int cols, const void* stage) {
    if (stage == nullptr || cols <= 0 || v.m % cols != 0) return 0;
    const long long ncol = static_cast<long long>(v.m_loc) * v.m;
    if ((ncol & (ncol - 1)) != 0 || ncol / cols > kMaxFusedLeaves || ncol / cols < 1) return 0;
    return static_cast<int>(ncol / cols);
}

// TMEM-resident sweep (k_thomas_tm). Shared memory is padded so that no more
// CTAs become resident on an SM than its 512 TMEM columns can serve (a CTA
// beyond that would only wait inside tcgen05.alloc).
template <typename T, bool Fast, bool Fused, class C>
int launch_thomas_tm_cfg(const SlabView<T>& v, T* r, const T* in, T* out, T* p2, T* pk,
                         Scalars<T>* S, const Scalars<T>* gate, T* stage, cudaStream_t st,
                         const Consume<T>* cs = nullptr) {
    const unsigned tcols = thomas_tm_cols(v.n_z, sizeof(T));
    const dim3 block(32, C::W);
    constexpr int PW = C::W / C::X;  // i-planes per CTA
    // Planes per CTA (X = 4): one TMEM allocation and profile load serve tpc
    // consecutive planes. The largest tpc <= 4 that keeps >= 6 waves of the 2
    // resident CTAs per SM with a last wave >= 97% full (C3: 4, K1 0.789 ->
    // 0.777 ms; tpc 3, 5, 6 leave a 24-62% last wave: 0.80-0.81 ms; 8: 0.855 ms).
    int tpc = 1;
    if (C::X == 4 && !v.halo.on) {
        const double slots = 2.0 * num_sms();
        const long long rows = (v.m + 127) / 128;
        for (int t = 4; t > 1; --t) {
            const double waves = static_cast<double>(rows * ((v.m_loc + t - 1) / t)) / slots;
            if (waves >= 6.0 && waves / std::ceil(waves) >= 0.97) {
                tpc = t;
                break;
            }
        }
    }
    const dim3 grid((v.m + 32 * C::X - 1) / (32 * C::X),
                    C::X == 4 ? (v.m_loc + tpc - 1) / tpc : (v.m_loc + PW - 1) / PW);
    size_t smem = thomas_tm_smem_bytes<T, C>(v.n_z);
    const size_t max_ctas = 512u / tcols;
    const size_t floor_bytes = 233472u / (max_ctas + 1) - 1024u + 64u;
    if (smem < floor_bytes) smem = floor_bytes;
    // fused stage 1: CTA = one aligned node (128 consecutive columns) of the tree
    const int leaves = fused_leaves(v, C::X == 4 ? C::NT : 0, Fused ? stage : nullptr);
    if constexpr (Fused && sizeof(T) == 8) {
        if (cs != nullptr) {
            if (!leaves) {
                std::fprintf(stderr, "acg: consumed reduction without fused K1 leaves\n");
                std::abort();
            }
            ensure_smem(k_thomas_tm<T, Fast, Fused, C, true>, smem);
            launch_pdl(k_thomas_tm<T, Fast, Fused, C, true>, grid, block, smem, st, v, r, in, out,
                       p2, pk, static_cast<const Scalars<T>*>(S), gate, tcols, stage, leaves, tpc,
                       *cs);
            return leaves;
        }
    }
    if (cs != nullptr) {
        std::fprintf(stderr, "acg: consumed reduction requested for an fp32 sweep\n");
        std::abort();
    }
    ensure_smem(k_thomas_tm<T, Fast, Fused, C>, smem);
    launch_pdl(k_thomas_tm<T, Fast, Fused, C>, grid, block, smem, st, v, r, in, out, p2, pk,
               static_cast<const Scalars<T>*>(S), gate, tcols, leaves ? stage : nullptr, leaves, tpc,
               Consume<T>{});
    return leaves;
}

// Two columns per thread, persistent (k_thomas_tm2); -1 if not applicable.
template <typename T, bool Fast, bool Fused, class C>
int launch_thomas_tm2_cfg(const SlabView<T>& v, T* r, const T* in, T* out, T* p2, T* pk,
                          Scalars<T>* S, const Scalars<T>* gate, T* stage, cudaStream_t st) {
    const unsigned tcols = 2 * thomas_tm_cols(v.n_z, sizeof(T));
    if (v.m % 2 != 0 || tcols > 512) return -1;
    const int per_sm = static_cast<int>(512u / tcols);
    const int tiles_row = (v.m + C::COLS - 1) / C::COLS;
    const int ntiles = tiles_row * v.m_loc;
    const int grid = std::min(ntiles, num_sms() * per_sm);
    size_t smem = thomas_tm2_smem_bytes<T, C>(v.n_z);
    const size_t floor_bytes = 233472u / (per_sm + 1) - 1024u + 64u;
    if (smem < floor_bytes) smem = floor_bytes;
    const int leaves = fused_leaves(v, C::COLS, Fused ? stage : nullptr);
    ensure_smem(k_thomas_tm2<T, Fast, Fused, C>, smem);
    k_thomas_tm2<T, Fast, Fused, C><<<grid, dim3(32, C::W), smem, st>>>(
        v, r, in, out, p2, pk, S, gate, tcols, leaves ? stage : nullptr, leaves, ntiles, tiles_row);
    return leaves;
}

// K1/K4 kernel choice (measured):
//  * fp32: k_thomas_tm2, two columns per thread with both z' columns in TMEM
//    (C4: K1 1.51 vs 2.09 ms for one column per thread — the fp32 sweep moves
//    half the bytes per instruction); needs even m;
//  * fp64, and fp32 with odd m: k_thomas_tm, one column per thread, z' in TMEM
//    (C3: 0.78 ms; two columns per thread 0.99 ms);
//  * columns whose z' needs all 512 TMEM columns (fp64 128 < n_z <= 256) run
//    k_thomas_tm with one CTA per SM (1024^2 x 256: K1 2.10 vs 3.55 ms);
//  * k_thomas (z' through global memory) when the TMEM sweep cannot run: n_z*s
//    above 2 KiB, or division operand ranges that fail k_validate_tm.
// Measured-slower configurations (TMA-fed tiles, other ring depths and CTA
// shapes, occupancy caps) were removed after round 1; DESIGN.md keeps their numbers.
using ThomasTmDefault = ThomasTmCfg<4, 15, 15>;
using ThomasTm2Default = ThomasTm2Cfg<4, 15, 15>;

template <typename T, bool Fast, bool Fused>
int launch_thomas(const SlabView<T>& v, T* r, const T* in, T* out, T* p2, T* pk, Scalars<T>* S,
                  const Scalars<T>* gate, T* phi_scratch, T* stage, cudaStream_t st,
                  const Consume<T>* cs = nullptr) {
    const bool tmem = v.tm_ok && phi_scratch == nullptr;
    if (cs != nullptr && !(tmem && sizeof(T) == 8 && thomas_tm_cols(v.n_z, sizeof(T)) <= 512)) {
        std::fprintf(stderr, "acg: consumed reduction requested for a sweep without it\n");
        std::abort();
    }
    if (tmem && sizeof(T) == 4) {
        const int l = launch_thomas_tm2_cfg<T, Fast, Fused, ThomasTm2Default>(v, r, in, out, p2, pk,
                                                                             S, gate, stage, st);
        if (l >= 0) return l;
    }
    // up to 256 columns: two CTAs per SM; 512 (fp64 n_z <= 256, fp32 <= 512): one
    if (tmem && thomas_tm_cols(v.n_z, sizeof(T)) <= 512)
        return launch_thomas_tm_cfg<T, Fast, Fused, ThomasTmDefault>(v, r, in, out, p2, pk, S, gate,
                                                                    stage, st, cs);
    if (v.halo.on) {  // fused_halo_ok admits only the TMEM sweeps
        std::fprintf(stderr, "acg: fused halo requested for a sweep that cannot carry it\n");
        std::abort();
    }
    launch_thomas_cfg<T, Fast, Fused, typename ThomasOf<T>::type>(v, r, in, out, p2, pk, S, gate,
                                                                  phi_scratch, st);
    return 0;
}

}  // namespace

#include "acg_csr.cuh"

TreePlan make_tree_plan(long long n) {
    TreePlan p{};
    p.n = n;
    int d = 0;
    while (((n + (1LL << d) - 1) >> d) > 16) ++d;
    p.depth = d;
    p.nodes = 1 << d;
    p.threads = p.nodes < 256 ? p.nodes : 256;
    p.blocks = p.nodes / p.threads;
    return p;
}

size_t thomas_smem_per_block(int dsize, int n_z, bool global_phi) {
    return dsize == 4 ? thomas_smem_bytes<float, ThomasF32>(n_z, global_phi)
                      : thomas_smem_bytes<double, ThomasF64>(n_z, global_phi);
}

template <typename T>
bool validate_thomas_tm(const SlabView<T>& v, cudaStream_t st) {
    int* bad = nullptr;
    if (cudaMalloc(&bad, sizeof(int)) != cudaSuccess) return false;
    cudaMemsetAsync(bad, 0, sizeof(int), st);
    const long long ncol = static_cast<long long>(v.m_loc) * v.m;
    k_validate_tm<T><<<grid_1d(ncol, 128), 128, 0, st>>>(v, bad);
    post_launch("validate_tm");
    int h = 1;
    cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    const bool ok = cudaStreamSynchronize(st) == cudaSuccess && h == 0;
    cudaFree(bad);
    return ok;
}

template <typename T>
int launch_fused_prec(const SlabView<T>& v, bool fast, T* r, T* z, const T* q, T* part_r2,
                      T* part_k, Scalars<T>* S, T* phi_scratch, T* stage, cudaStream_t st,
                      const Consume<T>* cs) {
    const int leaves =
        fast ? launch_thomas<T, true, true>(v, r, q, z, part_r2, part_k, S, nullptr, phi_scratch,
                                            stage, st, cs)
             : launch_thomas<T, false, true>(v, r, q, z, part_r2, part_k, S, nullptr, phi_scratch,
                                             stage, st, cs);
    post_launch("fused_prec");
    return leaves;
}

template <typename T>
void launch_precondition(const SlabView<T>& v, bool fast, const T* y, T* x, Scalars<T>* S,
                         const Scalars<T>* gate, T* phi_scratch, cudaStream_t st) {
    if (fast)
        launch_thomas<T, true, false>(v, nullptr, y, x, nullptr, nullptr, S, gate, phi_scratch,
                                      nullptr, st);
    else
        launch_thomas<T, false, false>(v, nullptr, y, x, nullptr, nullptr, S, gate, phi_scratch,
                                       nullptr, st);
    post_launch("precondition");
}

// K2 kernel choice (measured): fp64 with even m
// k_fused_spmv_pair2 (two columns per thread, every stencil input in a 3-level
// cp.async ring, C3 K2 1.18 ms); fp32 with m % 4 == 0 k_fused_spmv_quad (four
// columns per thread, the same ring with 16-byte quads, C4 K2 2.37 ms), other
// even m k_fused_spmv_pair (neighbour rows loaded a level ahead); odd m
// k_fused_spmv_tile (shared z tiles). Power-of-two fp64 panels narrower than
// 512 columns split the levels over 512/m thread groups (k_fused_spmv_pair2
// <..., KS>, C1 33.2 -> 27.6 us per iteration), and small single-slab grids
// finish the previous sweep's reduction in the prologue (<..., CS>; the K1
// side in k_thomas_tm<..., CS>), DESIGN.md §5.3.
// Measured-slower kernels (one column per thread with plain or ring loads) and
// the other ring depths were removed after round 1.
inline bool spmv_pairs(int m) { return m % 2 == 0; }
// ACG_KSPLIT=0: narrow panels sweep every level in one thread (A/B)
inline bool kseg_off() {
    static const bool off = [] {
        const char* e = std::getenv("ACG_KSPLIT");
        return e && std::string(e) == "0";
    }();
    return off;
}

template <typename T>
bool fused_halo_ok(const SlabView<T>& v, bool fast, bool phi_in_hbm) {
    (void)fast;
    static const bool off = [] {  // ACG_FUSED_HALO=0: copy + signal kernels instead (A/B)
        const char* e = std::getenv("ACG_FUSED_HALO");
        return e && std::string(e) == "0";
    }();
    // producer: k_thomas_tm2 (fp32) or k_thomas_tm (fp64); consumer: k_fused_spmv_quad /
    // k_fused_spmv_pair (fp32) or k_fused_spmv_pair2 (fp64)
    const unsigned cols = thomas_tm_cols(v.n_z, sizeof(T));
    const bool k1 = sizeof(T) == 4 ? 2 * cols <= 512 : cols <= 512;
    return !off && v.tm_ok && !phi_in_hbm && k1 && spmv_pairs(v.m);
}

template <typename T>
bool consume_plan(const SlabView<T>& v, bool phi_in_hbm, int* leaves_k1, int* leaves_k2) {
    static const bool off = [] {  // ACG_CONSUME=0: reduction kernels after each sweep (A/B)
        const char* e = std::getenv("ACG_CONSUME");
        return e && std::string(e) == "0";
    }();
    if (off || sizeof(T) != 8 || v.halo.on || !v.tm_ok || phi_in_hbm || !spmv_pairs(v.m) ||
        thomas_tm_cols(v.n_z, sizeof(T)) > 512)
        return false;
    // the leaf counts launch_thomas_tm_cfg and launch_fused_spmv produce (k_thomas_tm:
    // 128-column nodes; k_fused_spmv_pair2: 512 columns, or a narrower power-of-two plane)
    constexpr int kCols = 2 * 32 * kStencilWarps;
    const bool narrow = v.m < kCols && v.m >= 64 && (v.m & (v.m - 1)) == 0;
    const int a = fused_leaves(v, ThomasTmDefault::NT, v.prof);
    const int b = fused_leaves(v, narrow ? v.m : kCols, v.prof);
    if (a < 1 || b < 1 || a > kConsumeMaxLeaves || b > kConsumeMaxLeaves) return false;
    *leaves_k1 = a;
    *leaves_k2 = b;
    return true;
}

template <typename T>
bool spmv_plane_ranges(const SlabView<T>& v, bool fast) {
    (void)fast;
    return spmv_pairs(v.m);
}

template <typename T>
int launch_fused_spmv(const SlabView<T>& v, bool fast, T* u, T* p, T* q, const T* z, T* part,
                      const Scalars<T>* S, T* stage, cudaStream_t st, const Consume<T>* cs) {
    int leaves = 0;
    const dim3 block(32, kStencilWarps);
    if (cs != nullptr && !(sizeof(T) == 8 && spmv_pairs(v.m) && stage != nullptr)) {
        std::fprintf(stderr, "acg: consumed reduction requested for a sweep without it\n");
        std::abort();
    }
    if (v.halo.on && !(spmv_pairs(v.m) && v.plane_count == 0)) {
        std::fprintf(stderr, "acg: fused halo requested for a stencil sweep that cannot carry it\n");
        std::abort();
    }
    if (spmv_pairs(v.m)) {
        constexpr int kCols = 2 * 32 * kStencilWarps;  // columns per CTA (one i-plane)
        // tree node per CTA: kCols columns, or the whole plane of a narrower
        // power-of-two panel (pair_node_sums)
        const bool narrow = v.m < kCols && v.m >= 64 && (v.m & (v.m - 1)) == 0;
        leaves = fused_leaves(v, narrow ? v.m : kCols, stage);
        T* stg = leaves ? stage : nullptr;
        const dim3 g2((v.m + kCols - 1) / kCols, v.plane_count ? v.plane_count : v.m_loc);
        if constexpr (sizeof(T) == 4) {
            if (v.m % 4 == 0) {  // four columns per thread (k_fused_spmv_quad)
                constexpr int kQ = 4 * 32 * kStencilWarps;
                const bool nq = v.m < kQ && v.m >= 64 && (v.m & (v.m - 1)) == 0;
                leaves = fused_leaves(v, nq ? v.m : kQ, stage);
                T* stq = leaves ? stage : nullptr;
                const dim3 g4((v.m + kQ - 1) / kQ, v.plane_count ? v.plane_count : v.m_loc);
                // ring depth 3 (one 8-warp CTA per SM: 112 KB of ring); C4 K2 2.374 ms =
                // 6.37 TB/s vs 2.512 ms for k_fused_spmv_pair; depth 2 with two CTAs: 2.60 ms
                constexpr int D = 3;
                const size_t smem = static_cast<size_t>((4 * v.n_z + 3) & ~3) * sizeof(T) +
                                    static_cast<size_t>(D + 1) * 7 * 32 * kStencilWarps * 16;
                if (fast) {
                    ensure_smem(k_fused_spmv_quad<true, D, 1>, smem);
                    launch_pdl(k_fused_spmv_quad<true, D, 1>, g4, block, smem, st, v, u, p, q, z,
                               part, S, stq, leaves);
                } else {
                    ensure_smem(k_fused_spmv_quad<false, D, 1>, smem);
                    launch_pdl(k_fused_spmv_quad<false, D, 1>, g4, block, smem, st, v, u, p, q, z,
                               part, S, stq, leaves);
                }
                post_launch("fused_spmv");
                return leaves;
            }
            // ring depth 2 (exact: at least 3 CTAs per SM)
            constexpr int D = 2;
            const size_t smem = sizeof(T) * (4 * static_cast<size_t>(v.n_z) +
                                             static_cast<size_t>(D + 1) * 4 * kCols);
            if (fast) {
                ensure_smem(k_fused_spmv_pair<T, true, D, 2>, smem);
                k_fused_spmv_pair<T, true, D, 2><<<g2, block, smem, st>>>(v, u, p, q, z, part, S,
                                                                         stg, leaves);
            } else {
                ensure_smem(k_fused_spmv_pair<T, false, D, 3>, smem);
                k_fused_spmv_pair<T, false, D, 3><<<g2, block, smem, st>>>(v, u, p, q, z, part, S,
                                                                          stg, leaves);
            }
        } else {
            // ring depth 3, at least 2 CTAs per SM
            constexpr int D = 3;
            const size_t smem = sizeof(T) * (4 * static_cast<size_t>(v.n_z) +
                                             static_cast<size_t>(D + 1) * 7 * kCols);
            // narrow panels with the fused reduction: 512/m level groups per plane
            // (KS), their products of levels past group 0's in shared memory
            int kseg = narrow && stg != nullptr ? kCols / v.m : 1;
            // (ring depth 3 as for wide panels; depth 5, one CTA per SM: C1 K2 slower)
            size_t smem_ks = smem;
            if (kseg > 1) {
                const int len = (v.n_z + kseg - 1) / kseg;
                smem_ks += sizeof(T) * static_cast<size_t>(v.n_z - len) * v.m;
                if (smem_ks > 232448 || kseg_off()) kseg = 1;
            }
            const Consume<T> none{};
            const Consume<T>& c2 = cs ? *cs : none;
            if (cs != nullptr && !leaves) {
                std::fprintf(stderr, "acg: consumed reduction without fused K2 leaves\n");
                std::abort();
            }
#define ACG_PAIR2(FAST, CSM, KSM)                                                               \
    do {                                                                                        \
        auto kern = k_fused_spmv_pair2<T, FAST, D, 2, CSM, KSM>;                                \
        const size_t sb = KSM ? smem_ks : smem;                                                 \
        ensure_smem(kern, sb);                                                                  \
        launch_pdl(kern, g2, block, sb, st, v, u, p, q, z, part, S, stg, leaves, c2, kseg);     \
    } while (0)
            const bool ks = kseg > 1, csm = cs != nullptr;
            if (fast) {
                if (csm && ks) ACG_PAIR2(true, true, true);
                else if (csm) ACG_PAIR2(true, true, false);
                else if (ks) ACG_PAIR2(true, false, true);
                else ACG_PAIR2(true, false, false);
            } else {
                if (csm && ks) ACG_PAIR2(false, true, true);
                else if (csm) ACG_PAIR2(false, true, false);
                else if (ks) ACG_PAIR2(false, false, true);
                else ACG_PAIR2(false, false, false);
            }
#undef ACG_PAIR2
        }
    } else {
        constexpr int D = 5;  // shared z-tile ring depth
        const dim3 grid((v.m + 31) / 32, (v.m_loc + kStencilWarps - 1) / kStencilWarps);
        const size_t smem = spmv_tile_smem_bytes<T, kStencilWarps>(v.n_z);
        if (fast) {
            ensure_smem(k_fused_spmv_tile<T, true, kStencilWarps, D>, smem);
            k_fused_spmv_tile<T, true, kStencilWarps, D><<<grid, block, smem, st>>>(v, u, p, q, z,
                                                                                  part, S);
        } else {
            ensure_smem(k_fused_spmv_tile<T, false, kStencilWarps, D>, smem);
            k_fused_spmv_tile<T, false, kStencilWarps, D><<<grid, block, smem, st>>>(v, u, p, q, z,
                                                                                   part, S);
        }
    }
    post_launch("fused_spmv");
    return leaves;
}

template <typename T>
void launch_apply(const SlabView<T>& v, bool fast, const T* x, T* y, const Scalars<T>* gate,
                  cudaStream_t st) {
    const dim3 block(32, kStencilWarps);
    const dim3 grid((v.m + 31) / 32, (v.m_loc + kStencilWarps - 1) / kStencilWarps);
    const size_t smem = sizeof(T) * 4 * static_cast<size_t>(v.n_z);
    if (fast) {
        ensure_smem(k_apply<T, true>, smem);
        k_apply<T, true><<<grid, block, smem, st>>>(v, x, y, gate);
    } else {
        ensure_smem(k_apply<T, false>, smem);
        k_apply<T, false><<<grid, block, smem, st>>>(v, x, y, gate);
    }
    post_launch("apply");
}

template <typename T>
void launch_residual_partials(const SlabView<T>& v, bool fast, const T* u, const T* f, T* part,
                              cudaStream_t st) {
    const dim3 block(32, kStencilWarps);
    const dim3 grid((v.m + 31) / 32, (v.m_loc + kStencilWarps - 1) / kStencilWarps);
    const size_t smem = sizeof(T) * 4 * static_cast<size_t>(v.n_z);
    if (fast) {
        ensure_smem(k_residual_partials<T, true>, smem);
        k_residual_partials<T, true><<<grid, block, smem, st>>>(v, u, f, part);
    } else {
        ensure_smem(k_residual_partials<T, false>, smem);
        k_residual_partials<T, false><<<grid, block, smem, st>>>(v, u, f, part);
    }
    post_launch("residual_partials");
}

template <typename T>
void launch_dot_partials(const SlabView<T>& v, const T* x, const T* y, T* part,
                         const Scalars<T>* gate, cudaStream_t st) {
    const dim3 block(32, 8);
    const dim3 grid((v.m + 31) / 32, (v.m_loc + 7) / 8);
    k_dot_partials<T><<<grid, block, 0, st>>>(v, x, y, part, gate);
    post_launch("dot_partials");
}

template <typename T>
void launch_axpy(long long n, T value, const T* coef, bool neg, const T* x, T* y,
                 const Scalars<T>* gate, cudaStream_t st) {
    k_axpy<T><<<grid_1d(n, 256), 256, 0, st>>>(n, value, coef, neg ? 1 : 0, x, y, gate);
    post_launch("axpy");
}

template <typename T>
void launch_scal(long long n, T value, const T* coef, T* x, const Scalars<T>* gate,
                 cudaStream_t st) {
    k_scal<T><<<grid_1d(n, 256), 256, 0, st>>>(n, value, coef, x, gate);
    post_launch("scal");
}

template <typename T>
void launch_copy(long long n, const T* x, T* y, const Scalars<T>* gate, cudaStream_t st) {
    k_copy<T><<<grid_1d(n, 256), 256, 0, st>>>(n, x, y, gate);
    post_launch("copy");
}

template <typename T>
void launch_fill(long long n, T value, T* x, cudaStream_t st) {
    k_fill<T><<<grid_1d(n, 256), 256, 0, st>>>(n, value, x);
    post_launch("fill");
}

template <typename T>
void launch_fill_random(const SlabView<T>& v, uint64_t seed, T* x, cudaStream_t st) {
    const long long n = static_cast<long long>(v.m_loc) * v.plane;
    k_fill_random<T><<<grid_1d(n, 256), 256, 0, st>>>(v, seed, x);
    post_launch("fill_random");
}

template <typename T>
void launch_tree_stage1(const TreePlan& plan, const T* in0, const T* in1, const T* in2, int nv,
                        T* stage, const Scalars<T>* gate, cudaStream_t st) {
    k_tree1<T><<<plan.blocks, plan.threads, 0, st>>>(plan.n, plan.depth, in0, in1, in2, nv, stage,
                                                     plan.blocks, gate);
    post_launch("tree1");
}

template <typename T>
bool launch_tree_stage2(const TreePlan& plan, const T* stage, int nv, T* gather, int slab,
                        bool finish, int nslabs, bool exact_tree, Scalars<T>* S, int op,
                        cudaStream_t st, const IpcPut<T>* put) {
    IpcPut<T> pp = put ? *put : IpcPut<T>{nullptr, nullptr, 0, 0, 0};
    const int nl = plan.blocks;  // power of two
    // k_tree2_wide (<= 8192 leaves; above, k_tree_mid first) for the sweeps' one or
    // two values; k_tree2_shfl for three values (<= 16384 leaves); k_tree2 beyond
    if (nv <= 2 && nl > 1024 * 8 && nl <= 1024 * 8 * 1024) {
        // more leaves than one CTA takes: aligned nodes of 8192 leaves first
        const int nb = nl / 8192;
        T* mid = const_cast<T*>(stage) + static_cast<long long>(nv) * nl;
        launch_pdl(k_tree_mid<T>, dim3(nb), dim3(1024), 0, st, nl, stage, nv, mid);
        post_launch("tree_mid");
        TreePlan p2 = plan;
        p2.blocks = nb;
        return launch_tree_stage2<T>(p2, mid, nv, gather, slab, finish, nslabs, exact_tree, S, op,
                                     st, put);
    }
    if (nv <= 2 && nl <= 1024 * 8) {
        const int c = nl > 1024 ? nl / 1024 : 1;
        const int nt = nl / c;
        const int f = finish ? 1 : 0, ex = exact_tree ? 1 : 0;
        switch (c) {
            case 1: launch_pdl(k_tree2_wide<T, 1>, dim3(1), dim3(nt), 0, st, nl, stage, nv, gather, slab, f, nslabs, ex, S, op, pp); break;
            case 2: launch_pdl(k_tree2_wide<T, 2>, dim3(1), dim3(nt), 0, st, nl, stage, nv, gather, slab, f, nslabs, ex, S, op, pp); break;
            case 4: launch_pdl(k_tree2_wide<T, 4>, dim3(1), dim3(nt), 0, st, nl, stage, nv, gather, slab, f, nslabs, ex, S, op, pp); break;
            default: launch_pdl(k_tree2_wide<T, 8>, dim3(1), dim3(nt), 0, st, nl, stage, nv, gather, slab, f, nslabs, ex, S, op, pp); break;
        }
        post_launch("tree2");
        return pp.wait != nullptr;
    }
    pp.wait = nullptr;  // the other stage-2 kernels only put; k_finish waits and combines
    if (nl <= 256 * 64) {
        const int c = nl > 256 ? nl / 256 : 1;
        const int nt = nl / c;
        const int f = finish ? 1 : 0, ex = exact_tree ? 1 : 0;
        switch (c) {
            case 1: launch_pdl(k_tree2_shfl<T, 1>, dim3(1), dim3(nt), 0, st, nl, stage, nv, gather, slab, f, nslabs, ex, S, op, pp); break;
            case 2: launch_pdl(k_tree2_shfl<T, 2>, dim3(1), dim3(nt), 0, st, nl, stage, nv, gather, slab, f, nslabs, ex, S, op, pp); break;
            case 4: launch_pdl(k_tree2_shfl<T, 4>, dim3(1), dim3(nt), 0, st, nl, stage, nv, gather, slab, f, nslabs, ex, S, op, pp); break;
            case 8: launch_pdl(k_tree2_shfl<T, 8>, dim3(1), dim3(nt), 0, st, nl, stage, nv, gather, slab, f, nslabs, ex, S, op, pp); break;
            case 16: launch_pdl(k_tree2_shfl<T, 16>, dim3(1), dim3(nt), 0, st, nl, stage, nv, gather, slab, f, nslabs, ex, S, op, pp); break;
            case 32: launch_pdl(k_tree2_shfl<T, 32>, dim3(1), dim3(nt), 0, st, nl, stage, nv, gather, slab, f, nslabs, ex, S, op, pp); break;
            default: launch_pdl(k_tree2_shfl<T, 64>, dim3(1), dim3(nt), 0, st, nl, stage, nv, gather, slab, f, nslabs, ex, S, op, pp); break;
        }
        post_launch("tree2");
        return false;
    }
    const int nt = nl < 1024 ? nl : 1024;
    k_tree2<T><<<1, nt, 0, st>>>(nl, stage, nv, gather, slab, finish ? 1 : 0, nslabs,
                                 exact_tree ? 1 : 0, S, op);
    post_launch("tree2");
    return false;
}

template <typename T>
void launch_finish(const T* gather, int nv, int nslabs, bool exact_tree, Scalars<T>* S, int op,
                   cudaStream_t st, const unsigned long long* wait_flags, unsigned long long seq) {
    k_finish<T><<<1, 1, 0, st>>>(gather, nv, nslabs, exact_tree ? 1 : 0, S, op, wait_flags, seq);
    post_launch("finish");
}

void launch_ipc_signal(unsigned long long* const* flags, int n, unsigned long long seq,
                       cudaStream_t st) {
    FlagPtrs fp{};
    for (int i = 0; i < n && i < 8; ++i) fp.f[i] = flags[i];
    k_ipc_signal<<<1, 1, 0, st>>>(fp, n < 8 ? n : 8, seq);
    post_launch("ipc_signal");
}

__global__ void k_snapshot(const unsigned long long* __restrict__ src,
                           unsigned long long* __restrict__ dst, int words) {
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = __ldcg(src + i);
}

void launch_snapshot(const void* src, void* dst_mapped, int words, cudaStream_t st) {
    k_snapshot<<<1, 32, 0, st>>>(static_cast<const unsigned long long*>(src),
                                 static_cast<unsigned long long*>(dst_mapped), words);
    post_launch("snapshot");
}

void launch_ipc_wait(const unsigned long long* flags, int n, unsigned long long need,
                     unsigned long long seq, cudaStream_t st) {
    k_ipc_wait<<<1, 1, 0, st>>>(flags, n, need, seq);
    post_launch("ipc_wait");
}


template <typename T>
void launch_transpose(const T* in, T* out, int nx, int ny, int nb, long long isy, long long isb,
                      long long osx, long long osb, cudaStream_t st) {
    const dim3 block(32, 8);
    const int gz = nb < 65535 ? nb : 65535;
    const dim3 grid((nx + 31) / 32, (ny + 31) / 32, gz);
    k_transpose<T><<<grid, block, 0, st>>>(in, out, nx, ny, nb, isy, isb, osx, osb);
    post_launch("transpose");
}

#define ACG_INSTANTIATE(T)                                                                      \
    template bool validate_thomas_tm<T>(const SlabView<T>&, cudaStream_t);                      \
    template int launch_fused_prec<T>(const SlabView<T>&, bool, T*, T*, const T*, T*, T*,       \
                                      Scalars<T>*, T*, T*, cudaStream_t, const Consume<T>*);    \
    template bool consume_plan<T>(const SlabView<T>&, bool, int*, int*);                        \
    template void launch_precondition<T>(const SlabView<T>&, bool, const T*, T*, Scalars<T>*,   \
                                         const Scalars<T>*, T*, cudaStream_t);                  \
    template bool spmv_plane_ranges<T>(const SlabView<T>&, bool);                               \
    template bool fused_halo_ok<T>(const SlabView<T>&, bool, bool);                              \
    template int launch_fused_spmv<T>(const SlabView<T>&, bool, T*, T*, T*, const T*, T*,       \
                                      const Scalars<T>*, T*, cudaStream_t, const Consume<T>*);  \
    template void launch_apply<T>(const SlabView<T>&, bool, const T*, T*, const Scalars<T>*,    \
                                  cudaStream_t);                                                \
    template void launch_residual_partials<T>(const SlabView<T>&, bool, const T*, const T*, T*, \
                                              cudaStream_t);                                    \
    template void launch_dot_partials<T>(const SlabView<T>&, const T*, const T*, T*,            \
                                         const Scalars<T>*, cudaStream_t);                      \
    template void launch_axpy<T>(long long, T, const T*, bool, const T*, T*, const Scalars<T>*, \
                                 cudaStream_t);                                                 \
    template void launch_scal<T>(long long, T, const T*, T*, const Scalars<T>*, cudaStream_t);  \
    template void launch_copy<T>(long long, const T*, T*, const Scalars<T>*, cudaStream_t);     \
    template void launch_fill<T>(long long, T, T*, cudaStream_t);                               \
    template void launch_fill_random<T>(const SlabView<T>&, uint64_t, T*, cudaStream_t);        \
    template void launch_tree_stage1<T>(const TreePlan&, const T*, const T*, const T*, int, T*, \
                                        const Scalars<T>*, cudaStream_t);                       \
    template bool launch_tree_stage2<T>(const TreePlan&, const T*, int, T*, int, bool, int,     \
                                        bool, Scalars<T>*, int, cudaStream_t, const IpcPut<T>*); \
    template void launch_finish<T>(const T*, int, int, bool, Scalars<T>*, int, cudaStream_t,    \
                                   const unsigned long long*, unsigned long long);              \
    template void launch_transpose<T>(const T*, T*, int, int, int, long long, long long,        \
                                      long long, long long, cudaStream_t);                      \
    template void launch_csr_assemble<T>(const SlabView<T>&, int, long long*, int*, T*, T*, T*, \
                                         T*, cudaStream_t);                                     \
    template void launch_csr_spmv<T>(const SlabView<T>&, const long long*, const int*, const T*, \
                                     const T*, T*, const Scalars<T>*, cudaStream_t);            \
    template void launch_csr_tridiag<T>(const SlabView<T>&, const T*, const T*, const T*,       \
                                        const T*, T*, T*, Scalars<T>*, const Scalars<T>*,       \
                                        cudaStream_t);

ACG_INSTANTIATE(double)
ACG_INSTANTIATE(float)

}  // namespace acg
