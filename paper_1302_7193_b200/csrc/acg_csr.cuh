// Matrix-explicit backend on the GPU: the reference's
// CsrBackend (solver.hpp:126-145) — the stencil stored as a CSR matrix
// (csr.hpp:18-26, assembled as in csr.hpp:92-124) and the preconditioner as
// stored tridiagonal blocks (csr.hpp:31-36, :144-170), driven by the same
// standard PCG loop. It exists to reproduce the paper's matrix-free vs
// matrix-explicit comparison on B200 and to keep
// backend="csr" a drop-in; the headline path never touches it.
//
// Storage is B200-native, the arithmetic the reference's:
//  * rows follow the device plane-major order (il*plane + k*m + j), so a warp's
//    32 rows are 32 consecutive j and their ~224 entries one contiguous range;
//  * the entries of a row are ordered by the CALLER's layout linear index
//    (csr.hpp:stencil_row sorts by it), which fixes the summation order of
//    spmv_csr (csr.hpp:127-141), so results match CsrBackend bit for bit for
//    either layout; column indices are device offsets from the slab's plane 0
//    (negative / past-the-end ones address the ghost planes the halo fills);
//  * dl/dd/du live in the plane-major field layout (coalesced per column
//    thread) instead of canonical column order; same values, same Thomas
//    recurrence as solve_tridiag_set (csr.hpp:175-221).
// Assembly runs on the device (values formed in T from the context's tables
// with the reference's association order).

namespace {

// Entries per row before row (k, j) of a plane whose i-plane has ci in-panel
// i-neighbours (closed form of the row-count prefix sum).
__device__ __forceinline__ long long csr_plane_offset(int k, int j, int m, int n_z, int ci) {
    const long long cj = m > 1 ? 2ll * (m - 1) : 0;  // sum over j of the j-neighbour count
    const long long sk = static_cast<long long>(k > 0 ? k - 1 : 0) + (k < n_z - 1 ? k : n_z - 1);
    const int ck = (k > 0) + (k + 1 < n_z);
    const long long sj = static_cast<long long>(j > 0 ? j - 1 : 0) + (j < m - 1 ? j : m - 1);
    return static_cast<long long>(k) * (static_cast<long long>(m) * (1 + ci) + cj) +
           static_cast<long long>(m) * sk + static_cast<long long>(j) * (1 + ci + ck) + sj;
}

// Entries in the planes [i0, i0 + il) of a slab.
__device__ __forceinline__ long long csr_slab_offset(int il, int i0, int m, int n_z) {
    const long long cj = m > 1 ? 2ll * (m - 1) : 0;
    const long long ck = n_z > 1 ? 2ll * (n_z - 1) : 0;
    const long long sci = 2ll * il - ((i0 == 0 && il > 0) ? 1 : 0) - ((i0 + il >= m) ? 1 : 0);
    return static_cast<long long>(il) * (static_cast<long long>(n_z) * (m + cj) + m * ck) +
           static_cast<long long>(n_z) * m * sci;
}

// One thread per row: row_ptr, the sorted entries, and dl/dd/du.
template <typename T>
__global__ void __launch_bounds__(256)
    k_csr_assemble(const SlabView<T> v, int horizontal, long long* __restrict__ row_ptr,
                   int* __restrict__ col_idx, T* __restrict__ vals, T* __restrict__ dl,
                   T* __restrict__ dd, T* __restrict__ du) {
    using A = Ar<T, false>;
    const int m = v.m, n_z = v.n_z;
    const long long n_loc = static_cast<long long>(v.m_loc) * v.plane;
    const long long ncol = static_cast<long long>(v.m_loc) * m;
    for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < n_loc;
         r += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int il = static_cast<int>(r / v.plane);
        const long long rem = r - static_cast<long long>(il) * v.plane;
        const int k = static_cast<int>(rem / m), j = static_cast<int>(rem - static_cast<long long>(k) * m);
        const int i = v.i0 + il;
        const bool hw = i > 0, he = i + 1 < m, hs = j > 0, hn = j + 1 < m, hd = k > 0,
                   hu = k + 1 < n_z;
        const long long at0 = csr_slab_offset(il, v.i0, m, n_z) +
                              csr_plane_offset(k, j, m, n_z, int(hw) + int(he));
        const long long ci = static_cast<long long>(il) * m + j;
        const T area = v.col[kColArea * ncol + ci], adiag = v.col[kColDiag * ncol + ci];
        const T dk = v.prof[kProfD * n_z + k];
        // stencil_row values (csr.hpp:stencil_row), formed in T left to right
        const T self = A::mul(A::sub(A::mul(v.prof[kProfS * n_z + k], area), adiag), dk);
        const T up = A::mul(A::mul(area, v.prof[kProfB * n_z + k]), dk);
        const T down = A::mul(A::mul(area, v.prof[kProfC * n_z + k]), dk);
        const T east = A::mul(v.col[kColE * ncol + ci], dk);
        const T west = A::mul(v.col[kColW * ncol + ci], dk);
        const T north = A::mul(v.col[kColN * ncol + ci], dk);
        const T south = A::mul(v.col[kColS * ncol + ci], dk);
        const long long pl = v.plane;
        long long at = at0;
        auto put = [&](bool has, long long off, T val) {
            if (!has) return;
            col_idx[at] = static_cast<int>(r + off);
            vals[at] = val;
            ++at;
        };
        if (!horizontal) {  // l = n_z (m i + j) + k: i-1, j-1, k-1, self, k+1, j+1, i+1
            put(hw, -pl, west);
            put(hs, -1, south);
            put(hd, -m, down);
            put(true, 0, self);
            put(hu, m, up);
            put(hn, 1, north);
            put(he, pl, east);
        } else {            // l = m (n_z j + k) + i: j-1, k-1, i-1, self, i+1, k+1, j+1
            put(hs, -1, south);
            put(hd, -m, down);
            put(hw, -pl, west);
            put(true, 0, self);
            put(he, pl, east);
            put(hu, m, up);
            put(hn, 1, north);
        }
        row_ptr[r] = at0;
        if (r == n_loc - 1) row_ptr[n_loc] = at;
        // TridiagonalSet (csr.hpp:144-170): dl 0 at k = 0, du 0 at k = n_z - 1
        dd[r] = self;
        du[r] = hu ? up : T(0);
        dl[r] = hd ? down : T(0);
    }
}

// y = A x, one thread per row (csr.hpp:127-141: sum from 0 in entry order).
template <typename T>
__global__ void __launch_bounds__(256)
    k_csr_spmv(long long n_loc, const long long* __restrict__ row_ptr,
               const int* __restrict__ col_idx, const T* __restrict__ vals,
               const T* __restrict__ x, T* __restrict__ y, const Scalars<T>* __restrict__ gate) {
    using A = Ar<T, false>;
    if (gate && gate->done) return;
    for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < n_loc;
         r += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long e0 = row_ptr[r], e1 = row_ptr[r + 1];
        T sum = T(0);
        for (long long e = e0; e < e1; ++e)
            sum = A::add(sum, A::mul(vals[e], x[col_idx[e]]));
        y[r] = sum;
    }
}

// x = M^-1 y with the stored tridiagonals, one thread per column
// (csr.hpp:175-221: phi, forward elimination, back substitution).
template <typename T>
__global__ void __launch_bounds__(128)
    k_csr_tridiag(const SlabView<T> v, const T* __restrict__ dl, const T* __restrict__ dd,
                  const T* __restrict__ du, const T* __restrict__ y, T* __restrict__ x,
                  T* __restrict__ phi, Scalars<T>* flag, const Scalars<T>* __restrict__ gate) {
    using A = Ar<T, false>;
    if (gate && gate->done) return;
    const int m = v.m, n_z = v.n_z;
    const long long ncol = static_cast<long long>(v.m_loc) * m;
    const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (c >= ncol) return;
    const int il = static_cast<int>(c / m), j = static_cast<int>(c - static_cast<long long>(il) * m);
    const long long base = static_cast<long long>(il) * v.plane + j;
    T diag = dd[base];
    if (diag == T(0)) {
        flag->pivot = 2;
        return;
    }
    T ph = A::div(du[base], diag);
    phi[base] = ph;
    T xp = A::div(y[base], diag);
    x[base] = xp;
    long long l = base;
    for (int k = 1; k < n_z; ++k) {
        l += m;
        const T dlk = dl[l];
        diag = A::sub(dd[l], A::mul(dlk, ph));
        if (diag == T(0)) {
            flag->pivot = 2;
            return;
        }
        ph = A::div(du[l], diag);
        phi[l] = ph;
        xp = A::div(A::sub(y[l], A::mul(dlk, xp)), diag);
        x[l] = xp;
    }
    for (int k = n_z - 2; k >= 0; --k) {
        l -= m;
        xp = A::sub(x[l], A::mul(phi[l], xp));
        x[l] = xp;
    }
}

}  // namespace

template <typename T>
void launch_csr_assemble(const SlabView<T>& v, int horizontal, long long* row_ptr, int* col_idx,
                         T* vals, T* dl, T* dd, T* du, cudaStream_t st) {
    const long long n = static_cast<long long>(v.m_loc) * v.plane;
    k_csr_assemble<T><<<grid_1d(n, 256), 256, 0, st>>>(v, horizontal, row_ptr, col_idx, vals, dl,
                                                        dd, du);
    post_launch("csr_assemble");
}

template <typename T>
void launch_csr_spmv(const SlabView<T>& v, const long long* row_ptr, const int* col_idx,
                     const T* vals, const T* x, T* y, const Scalars<T>* gate, cudaStream_t st) {
    const long long n = static_cast<long long>(v.m_loc) * v.plane;
    k_csr_spmv<T><<<grid_1d(n, 256), 256, 0, st>>>(n, row_ptr, col_idx, vals, x, y, gate);
    post_launch("csr_spmv");
}

template <typename T>
void launch_csr_tridiag(const SlabView<T>& v, const T* dl, const T* dd, const T* du, const T* y,
                        T* x, T* phi, Scalars<T>* flag, const Scalars<T>* gate, cudaStream_t st) {
    const long long ncol = static_cast<long long>(v.m_loc) * v.m;
    k_csr_tridiag<T><<<static_cast<unsigned>((ncol + 127) / 128), 128, 0, st>>>(
        v, dl, dd, du, y, x, phi, flag, gate);
    post_launch("csr_tridiag");
}
