// K2 with the stencil input staged as shared-memory tiles (included by
// acg_kernels.cu after the K2/K3 definitions).
//
//   k_fused_spmv_tile   interleaved_spmv_kernel   operator.hpp:214-266 (Alg. 2)
//
// k_fused_spmv_ring streams p, q, u and z(k+1) through a per-thread cp.async
// ring but reads the four horizontal z neighbours with plain loads; those L1/L2
// round trips sit on every level's critical path and were the dominant stall
// (ncu: one DMUL waiting on them held half the warp samples). Here a CTA of
// W warps (W i-planes x 32 j) copies, for every level, the z tile it needs
// including a one-cell halo, (W+2) x 34 values, into a shared ring D levels
// ahead; every neighbour is then a shared-memory load. A CTA barrier per level
// publishes the tile (each value is copied by one thread and read by up to
// five). DRAM traffic is unchanged (halo rows come from L2): u, p, q R+W, z R.
// Arithmetic and association are those of k_fused_spmv (bit-identical).
template <int W>
struct SpmvTile {
    static constexpr int R = W + 2, CW = 34, N = R * CW, NT = 32 * W, NS = 8;
};

template <typename T, int W>
__host__ __device__ constexpr size_t spmv_tile_smem_bytes(int n_z) {
    using G = SpmvTile<W>;
    return sizeof(T) * (4 * static_cast<size_t>(n_z) + static_cast<size_t>(G::NS) * 3 * G::NT +
                        static_cast<size_t>(G::NS) * G::N);
}

template <typename T, bool Fast, int W, int D>
__global__ void __launch_bounds__(32 * W)
    k_fused_spmv_tile(const SlabView<T> v, T* __restrict__ u, T* __restrict__ p,
                      T* __restrict__ q, const T* __restrict__ z, T* __restrict__ part,
                      const Scalars<T>* __restrict__ S) {
    using A = Ar<T, Fast>;
    using G = SpmvTile<W>;
    constexpr int NT = G::NT, NS = G::NS, CW = G::CW, TN = G::N;
    static_assert(D >= 1 && D <= NS - 2, "the tile of level k+D+1 reuses the slot of level k-1");
    static_assert(W >= 4 && W + 2 <= 32, "four warps load the halo");
    if (S->done) return;  // block-uniform
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* prof = reinterpret_cast<T*>(smem_raw);
    const int n_z = v.n_z, m = v.m;
    const int lane = threadIdx.x, w = threadIdx.y;
    const int tid = w * 32 + lane;
    load_profile(prof, v.prof, 4 * n_z, tid, NT);
    T* ring = prof + 4 * n_z + tid;  // [slot][3][NT]: p, q, u
    T* tile = prof + 4 * n_z + NS * 3 * NT;  // [slot][R][CW]
    const T* sP = prof + kProfS * n_z;
    const T* bP = prof + kProfB * n_z;
    const T* cP = prof + kProfC * n_z;
    const T* dP = prof + kProfD * n_z;

    const int j0 = blockIdx.x * 32, il0 = blockIdx.y * W;
    const int j = j0 + lane, il = il0 + w;
    const bool valid = j < m && il < v.m_loc;
    const int jc = j < m ? j : m - 1;
    const int ilc = il < v.m_loc ? il : v.m_loc - 1;
    const Col<T> c = load_col(v, ilc, jc);
    // tile coordinates of this column and of its four neighbours (a missing
    // neighbour reads the column's own value with coefficient 0, operator.hpp:85-92)
    const int own = (w + 1) * CW + lane + 1;
    const int oe = c.oe != 0 ? CW : 0, ow = c.ow != 0 ? -CW : 0;
    const int on = c.on != 0 ? 1 : 0, os = c.os != 0 ? -1 : 0;
    // tile loads: every thread copies the value at its own tile position; warps
    // 0/1 also copy halo rows 0 / W+1, warps 2/3 (lanes < W+2) halo columns 0 / 33.
    // Rows outside the slab clamp to its ghost planes, columns to [0, m).
    auto gaddr = [&](int rr, int cc) -> const T* {
        int it = il0 - 1 + rr;
        it = it < -1 ? -1 : (it > v.m_loc ? v.m_loc : it);
        int jt = j0 - 1 + cc;
        jt = jt < 0 ? 0 : (jt >= m ? m - 1 : jt);
        return z + static_cast<long long>(it) * v.plane + jt;
    };
    const T* g0 = gaddr(w + 1, lane + 1);
    const T* g1 = nullptr;
    int s1 = 0;
    if (w == 0) {
        g1 = gaddr(0, lane + 1);
        s1 = lane + 1;
    } else if (w == 1) {
        g1 = gaddr(W + 1, lane + 1);
        s1 = (W + 1) * CW + lane + 1;
    } else if (w == 2 && lane < W + 2) {
        g1 = gaddr(lane, 0);
        s1 = lane * CW;
    } else if (w == 3 && lane < W + 2) {
        g1 = gaddr(lane, CW - 1);
        s1 = lane * CW + CW - 1;
    }
    const long long base = static_cast<long long>(ilc) * v.plane + jc;
    T* uc = u + base;
    T* pc = p + base;
    T* qc = q + base;
    const long long sm = m;

    auto issue_tile = [&](int kk, int slot) {  // z tile of level kk into tile slot
        T* ts = tile + slot * TN;
        cpa(ts + own, g0 + kk * sm);
        if (g1) cpa(ts + s1, g1 + kk * sm);
    };
    auto issue = [&](int kk, int slot) {  // level kk: p, q, u and the z tile of kk+1
        cpa(ring + (3 * slot + 0) * NT, pc + kk * sm);
        cpa(ring + (3 * slot + 1) * NT, qc + kk * sm);
        cpa(ring + (3 * slot + 2) * NT, uc + kk * sm);
        if (kk + 1 < n_z) issue_tile(kk + 1, (slot + 1) & (NS - 1));
    };
    issue_tile(0, 0);
    cp_commit();
#pragma unroll
    for (int t = 0; t < D; ++t) {
        if (t < n_z) issue(t, t);
        cp_commit();
    }
    __syncthreads();  // profile
    const T alpha = S->alpha, beta = S->beta;
    T zd = T(0), sig = T(0);
    for (int kg = 0; kg < n_z; kg += NS) {
#pragma unroll
        for (int t = 0; t < NS; ++t) {
            const int k = kg + t;
            if (k < n_z) {  // block-uniform
                cp_wait<D - 1>();
                __syncthreads();
                const T* ts = tile + t * TN;
                const T z0 = ts[own];
                if (k == 0) zd = z0;
                const T zu = k + 1 < n_z ? tile[((t + 1) & (NS - 1)) * TN + own] : z0;
                const T ze = ts[own + oe], zw = ts[own + ow], zn = ts[own + on], zs = ts[own + os];
                T pv = ring[(3 * t + 0) * NT], qv = ring[(3 * t + 1) * NT];
                const T uv = ring[(3 * t + 2) * NT];
                if (k + D < n_z) issue(k + D, (t + D) & (NS - 1));
                cp_commit();
                const long long l = static_cast<long long>(k) * sm;
                const T un = A::add(uv, A::mul(alpha, pv));
                pv = A::add(A::mul(beta, pv), z0);
                qv = A::mul(beta, qv);
                const T dq = stencil<T, Fast>(sP[k], c.area, c.adiag, bP[k], cP[k], c.ae, c.aw,
                                              c.an, c.as, z0, zu, zd, ze, zw, zn, zs);
                qv = A::add(qv, A::mul(dP[k], dq));
                sig = A::add(sig, A::mul(pv, qv));
                if (valid) {
                    __stcs(uc + l, un);
                    __stcs(pc + l, pv);
                    __stcs(qc + l, qv);
                }
                zd = z0;
            }
        }
    }
    cp_wait<0>();
    if (valid) part[static_cast<long long>(il) * m + j] = sig;
}



__device__ __forceinline__ void st_pair_cs(double* a, const Pair<double>& v) {
    __stcs(reinterpret_cast<double2*>(a), make_double2(v.x, v.y));
}
__device__ __forceinline__ void st_pair_cs(float* a, const Pair<float>& v) {
    __stcs(reinterpret_cast<float2*>(a), make_float2(v.x, v.y));
}

// Fused reduction stage 1 of the pair sweeps: the CTA's columns [j0, j0 + CW)
// of plane il (CW = 2 NT = 512) are one node of the pairwise tree; a narrower
// power-of-two panel (m < CW) makes the plane's m columns the node instead, so
// small grids keep the fused reduction (no k_tree1 launch). `red` holds the
// CTA's column partials in column order.
template <typename T, int CW>
__device__ __forceinline__ void pair_node_sums(const T* red, T* stage, int nleaves, int il, int m) {
    if (m >= CW) {
        cta_subtree_sums<T, CW>(red, 1, stage, nleaves,
                                (static_cast<long long>(il) * m + blockIdx.x * CW) / CW);
        return;
    }
    switch (m) {  // blockIdx.x == 0: the node is the whole plane
        case 256: cta_subtree_sums<T, 256>(red, 1, stage, nleaves, il); break;
        case 128: cta_subtree_sums<T, 128>(red, 1, stage, nleaves, il); break;
        default: cta_subtree_sums<T, 64>(red, 1, stage, nleaves, il); break;
    }
}

// K2 with two adjacent columns per thread (default for fp32): every stream
// moves the pair as one 8-byte (fp32) / 16-byte (fp64) vector, so the
// per-thread bookkeeping is paid once per two columns. CTA = one i-plane x
// 512 j. Column j's north neighbour is the pair's .y and column j+1's south
// neighbour its .x; only z(j-1) and z(j+2) come from outside the pair.
template <typename T, bool Fast, int D, int MINB>
__global__ void __launch_bounds__(32 * kStencilWarps, MINB)
    k_fused_spmv_pair(const SlabView<T> v, T* __restrict__ u, T* __restrict__ p,
                      T* __restrict__ q, const T* __restrict__ z, T* __restrict__ part,
                      const Scalars<T>* __restrict__ S, T* __restrict__ stage, int nleaves) {
    using A = Ar<T, Fast>;
    using P = Pair<T>;
    constexpr int NT = 32 * kStencilWarps, NS = D + 1;
    if (S->done) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* prof = reinterpret_cast<T*>(smem_raw);
    const int n_z = v.n_z, m = v.m;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    load_profile(prof, v.prof, 4 * n_z, tid, NT);
    __syncthreads();
    int il = v.plane_begin + blockIdx.y;
    if (v.halo.on) {  // fused halo: boundary planes last, after the neighbours' K1 put them
        const int y = blockIdx.y, ml = v.m_loc;
        if (ml >= 3) il = y < ml - 2 ? y + 1 : (y == ml - 2 ? 0 : ml - 1);
        if (il == 0 && v.halo.ghost[0] != nullptr) halo_acquire(v.halo.wait_flag[0], v.halo.seq);
        if (il == ml - 1 && v.halo.ghost[1] != nullptr) halo_acquire(v.halo.wait_flag[1], v.halo.seq);
    }
    const int jr = blockIdx.x * 2 * NT + 2 * tid;
    const bool valid = jr < m;  // m even: both columns exist
    if (stage == nullptr && !valid) return;
    const int j = valid ? jr : m - 2;
    P* ring = reinterpret_cast<P*>(prof + 4 * n_z) + tid;  // [slot][4][NT]
    const T* sP = prof + kProfS * n_z;
    const T* bP = prof + kProfB * n_z;
    const T* cP = prof + kProfC * n_z;
    const T* dP = prof + kProfD * n_z;
    const Col<T> ca = load_col(v, il, j);
    const Col<T> cb = load_col(v, il, j + 1);
    const T alpha = S->alpha, beta = S->beta;
    const long long base = static_cast<long long>(il) * v.plane + j;
    const T* zc = z + base;
    T* uc = u + base;
    T* pc = p + base;
    T* qc = q + base;
    const long long sm = m;
    T siga = T(0), sigb = T(0);
    if (valid) {  // the idle warps of a narrow panel's CTA (fused reduction) skip the sweep
        auto issue = [&](int k, int s) {
            const long long l = static_cast<long long>(k) * sm;
            P* r0 = ring + s * 4 * NT;
            cpa_pair<T>(r0, pc + l);
            cpa_pair<T>(r0 + NT, qc + l);
            cpa_pair<T>(r0 + 2 * NT, uc + l);
            if (k + 1 < n_z) cpa_pair<T>(r0 + 3 * NT, zc + l + sm);
        };
    #pragma unroll
        for (int t = 0; t < D; ++t) {
            if (t < n_z) issue(t, t);
            cp_commit();
        }
        P z0 = *reinterpret_cast<const P*>(zc), zd = z0;
        // outside neighbours one level ahead: i+-1 rows as pairs, z(j-1), z(j+2)
        long long oe = ca.oe, ow = ca.ow;  // same for both columns (same plane)
        if (v.halo.on) {  // ghost rows straight from this rank's mailbox
            if (il == 0 && v.halo.ghost[0] != nullptr) ow = (v.halo.ghost[0] + j) - zc;
            if (il == v.m_loc - 1 && v.halo.ghost[1] != nullptr) oe = (v.halo.ghost[1] + j) - zc;
        }
        // i+-1 rows through L2 (coherent: the ghost rows may be a peer's fresh stores)
        P ze = ldcg_pair<T>(zc + oe), zw = ldcg_pair<T>(zc + ow);
        T zs = zc[ca.os], zn = zc[1 + cb.on];
        int cs = 0, ps_ = D;
        for (int k = 0; k < n_z; ++k) {
            const long long l = static_cast<long long>(k) * sm;
            const P ce = ze, cw = zw;
            const T cs0 = zs, cn1 = zn;
            if (k + 1 < n_z) {
                const long long l1 = l + sm;
                ze = ldcg_pair<T>(zc + l1 + oe);
                zw = ldcg_pair<T>(zc + l1 + ow);
                zs = zc[l1 + ca.os];
                zn = zc[l1 + 1 + cb.on];
            }
            cp_wait<D - 1>();
            const P* r0 = ring + cs * 4 * NT;
            P pv = r0[0], qv = r0[NT];
            const P uv = r0[2 * NT];
            const P zu = k + 1 < n_z ? r0[3 * NT] : z0;
            if (k + D < n_z) issue(k + D, ps_);
            cp_commit();
            cs = cs + 1 == NS ? 0 : cs + 1;
            ps_ = ps_ + 1 == NS ? 0 : ps_ + 1;
            const P un{A::add(uv.x, A::mul(alpha, pv.x)), A::add(uv.y, A::mul(alpha, pv.y))};
            pv.x = A::add(A::mul(beta, pv.x), z0.x);
            pv.y = A::add(A::mul(beta, pv.y), z0.y);
            qv.x = A::mul(beta, qv.x);
            qv.y = A::mul(beta, qv.y);
            // column j: north = own .y (exists: m even), south = z(j-1) (own value on the edge)
            const T dqa = stencil<T, Fast>(sP[k], ca.area, ca.adiag, bP[k], cP[k], ca.ae, ca.aw, ca.an,
                                           ca.as, z0.x, zu.x, zd.x, ce.x, cw.x, z0.y, cs0);
            // column j+1: south = own .x, north = z(j+2) (own value on the edge)
            const T dqb = stencil<T, Fast>(sP[k], cb.area, cb.adiag, bP[k], cP[k], cb.ae, cb.aw, cb.an,
                                           cb.as, z0.y, zu.y, zd.y, ce.y, cw.y, cn1, z0.x);
            qv.x = A::add(qv.x, A::mul(dP[k], dqa));
            qv.y = A::add(qv.y, A::mul(dP[k], dqb));
            siga = A::add(siga, A::mul(pv.x, qv.x));
            sigb = A::add(sigb, A::mul(pv.y, qv.y));
            if (valid) {
                st_pair_cs(uc + l, un);
                st_pair_cs(pc + l, pv);
                st_pair_cs(qc + l, qv);
            }
            zd = z0;
            z0 = zu;
        }
        cp_wait<0>();
    }
    if (stage != nullptr) {  // fused reduction stage 1: the CTA's 512 columns are a tree node
        __syncthreads();
        T* red = prof + 4 * n_z;
        red[2 * tid] = siga;
        red[2 * tid + 1] = sigb;
        __syncthreads();
        if (threadIdx.y == 0)
            pair_node_sums<T, 2 * NT>(red, stage, nleaves, il, m);
        return;
    }
    *reinterpret_cast<P*>(part + static_cast<long long>(il) * m + j) = P{siga, sigb};
}

// CS: consumed-reduction mode — the prologue finishes the previous K1's
// reduction (consume_finish) instead of reading alpha, beta and done from S.
// KS: level split for narrow panels (CTA = one plane of m < 512 columns, so only
// m/2 of the 256 threads would hold a column pair): kseg = 512/m groups of m/2
// threads sweep consecutive level ranges of the same columns — every level's
// u, p, q are independent of the others, only the vertical neighbours z(k-1),
// z(k+1) cross a range boundary and are plain loads. <p, q> stays the
// reference's sequential sum over k (operator.hpp:395-404): group 0 sums its
// levels on the fly, groups >= 1 park their products in shared memory, and
// group 0 continues the same running sum through them in level order.
template <typename T, bool Fast, int D, int MINB, bool CS = false, bool KS = false>
__global__ void __launch_bounds__(32 * kStencilWarps, MINB)
    k_fused_spmv_pair2(const SlabView<T> v, T* __restrict__ u, T* __restrict__ p,
                      T* __restrict__ q, const T* __restrict__ z, T* __restrict__ part,
                      const Scalars<T>* __restrict__ S, T* __restrict__ stage, int nleaves,
                      const Consume<T> cs, int kseg) {
    using A = Ar<T, Fast>;
    using P = Pair<T>;
    constexpr int NT = 32 * kStencilWarps, NS = D + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* prof = reinterpret_cast<T*>(smem_raw);
    const int n_z = v.n_z, m = v.m;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    load_profile(prof, v.prof, 4 * n_z, tid, NT);  // static data: before the dependency wait
    __syncthreads();
    pdl_wait();  // programmatic dependent launch: the previous grid has completed
    T alpha = T(0), beta = T(0);
    if constexpr (!CS) {
        if (ld_dep(&S->done)) return;  // block-uniform
    }
    int il = v.plane_begin + blockIdx.y;
    if (v.halo.on) {  // fused halo: boundary planes last, after the neighbours' K1 put them
        const int y = blockIdx.y, ml = v.m_loc;
        if (ml >= 3) il = y < ml - 2 ? y + 1 : (y == ml - 2 ? 0 : ml - 1);
        if (il == 0 && v.halo.ghost[0] != nullptr) halo_acquire(v.halo.wait_flag[0], v.halo.seq);
        if (il == ml - 1 && v.halo.ghost[1] != nullptr) halo_acquire(v.halo.wait_flag[1], v.halo.seq);
    }
    int jr = blockIdx.x * 2 * NT + 2 * tid;
    int grp = 0, k0 = 0, k1 = n_z;  // KS: this thread's level group and range
    if constexpr (KS) {
        const int half = m >> 1;  // column pairs per plane; kseg * half == NT
        grp = tid / half;
        jr = 2 * (tid - grp * half);
        const int len = (n_z + kseg - 1) / kseg;
        k0 = min(n_z, grp * len);
        k1 = min(n_z, k0 + len);
    }
    const bool valid = jr < m;  // m even: both columns exist
    if (stage == nullptr && !valid) return;
    const int j = valid ? jr : m - 2;
    P* ring = reinterpret_cast<P*>(prof + 4 * n_z) + tid;  // [slot][7][NT] (6 pairs + 2 edge scalars)
    // KS: products of levels [len, n_z) as pairs [k - len][m / 2], after the ring
    P* prod = reinterpret_cast<P*>(prof + 4 * n_z) + NS * 7 * NT;
    const T* sP = prof + kProfS * n_z;
    const T* bP = prof + kProfB * n_z;
    const T* cP = prof + kProfC * n_z;
    const T* dP = prof + kProfD * n_z;
    const Col<T> ca = load_col(v, il, j);
    const Col<T> cb = load_col(v, il, j + 1);
    if constexpr (!CS) {
        alpha = ld_dep(&S->alpha);
        beta = ld_dep(&S->beta);
    }
    const long long base = static_cast<long long>(il) * v.plane + j;
    const T* zc = z + base;
    T* uc = u + base;
    T* pc = p + base;
    T* qc = q + base;
    const long long sm = m;
    T siga = T(0), sigb = T(0);
    long long oe = ca.oe, ow = ca.ow;  // same for both columns (same plane)
    if (v.halo.on) {  // ghost rows straight from this rank's mailbox
        if (il == 0 && v.halo.ghost[0] != nullptr) ow = (v.halo.ghost[0] + j) - zc;
        if (il == v.m_loc - 1 && v.halo.ghost[1] != nullptr) oe = (v.halo.ghost[1] + j) - zc;
    }
    {
        auto issue = [&](int k, int s) {
            const long long l = static_cast<long long>(k) * sm;
            P* r0 = ring + s * 7 * NT;
            cpa_pair<T>(r0, pc + l);
            cpa_pair<T>(r0 + NT, qc + l);
            cpa_pair<T>(r0 + 2 * NT, uc + l);
            if (k + 1 < n_z) cpa_pair<T>(r0 + 3 * NT, zc + l + sm);
            cpa_pair<T>(r0 + 4 * NT, zc + l + oe);
            cpa_pair<T>(r0 + 5 * NT, zc + l + ow);
            T* e = reinterpret_cast<T*>(r0 + 6 * NT);  // z(j-1), z(j+2) (own values on the edges)
            cpa(e, zc + l + ca.os);
            cpa(e + 1, zc + l + 1 + cb.on);
        };
        // the idle warps of a narrow panel's CTA (fused reduction) skip the sweep
    #pragma unroll
        for (int t = 0; t < D; ++t) {
            if (valid && k0 + t < k1) issue(k0 + t, t);
            cp_commit();
        }
        if constexpr (CS) {  // the previous reduction's finish while the ring fills
            __shared__ T cs_red[64];
            const Consumed<T> cr = consume_finish<T, NT>(cs, tid, cs_red);
            if (cr.done) {  // block-uniform
                cp_wait<0>();
                return;
            }
            alpha = cr.alpha;
            beta = cr.beta;
        }
        if (valid) {
            P z0{T(0), T(0)}, zd{T(0), T(0)};
            if (k0 < k1) {
                z0 = *reinterpret_cast<const P*>(zc + static_cast<long long>(k0) * sm);
                zd = k0 > 0 ? *reinterpret_cast<const P*>(zc + static_cast<long long>(k0 - 1) * sm) : z0;
            }
            const int len = KS ? (n_z + kseg - 1) / kseg : 0;  // KS: group 0's level count
            int cur = 0, ps_ = D;
            for (int k = k0; k < k1; ++k) {
                const long long l = static_cast<long long>(k) * sm;
                cp_wait<D - 1>();
                const P* r0 = ring + cur * 7 * NT;
                P pv = r0[0], qv = r0[NT];
                const P uv = r0[2 * NT];
                const P zu = k + 1 < n_z ? r0[3 * NT] : z0;
                const P ce = r0[4 * NT], cw = r0[5 * NT];
                const P ex = r0[6 * NT];
                const T cs0 = ex.x, cn1 = ex.y;
                if (k + D < k1) issue(k + D, ps_);
                cp_commit();
                cur = cur + 1 == NS ? 0 : cur + 1;
                ps_ = ps_ + 1 == NS ? 0 : ps_ + 1;
                const P un{A::add(uv.x, A::mul(alpha, pv.x)), A::add(uv.y, A::mul(alpha, pv.y))};
                pv.x = A::add(A::mul(beta, pv.x), z0.x);
                pv.y = A::add(A::mul(beta, pv.y), z0.y);
                qv.x = A::mul(beta, qv.x);
                qv.y = A::mul(beta, qv.y);
                // column j: north = own .y (exists: m even), south = z(j-1) (own value on the edge)
                const T dqa = stencil<T, Fast>(sP[k], ca.area, ca.adiag, bP[k], cP[k], ca.ae, ca.aw, ca.an,
                                               ca.as, z0.x, zu.x, zd.x, ce.x, cw.x, z0.y, cs0);
                // column j+1: south = own .x, north = z(j+2) (own value on the edge)
                const T dqb = stencil<T, Fast>(sP[k], cb.area, cb.adiag, bP[k], cP[k], cb.ae, cb.aw, cb.an,
                                               cb.as, z0.y, zu.y, zd.y, ce.y, cw.y, cn1, z0.x);
                qv.x = A::add(qv.x, A::mul(dP[k], dqa));
                qv.y = A::add(qv.y, A::mul(dP[k], dqb));
                if (KS && grp > 0) {
                    prod[(k - len) * (m >> 1) + (j >> 1)] = P{A::mul(pv.x, qv.x), A::mul(pv.y, qv.y)};
                } else {
                    siga = A::add(siga, A::mul(pv.x, qv.x));
                    sigb = A::add(sigb, A::mul(pv.y, qv.y));
                }
                if (valid) {
                    st_pair_cs(uc + l, un);
                    st_pair_cs(pc + l, pv);
                    st_pair_cs(qc + l, qv);
                }
                zd = z0;
                z0 = zu;
            }
            cp_wait<0>();
        }
    }
    if constexpr (KS) {  // group 0 carries the running sums through the later levels
        __syncthreads();
        if (grp == 0) {
            const int len = (n_z + kseg - 1) / kseg;
            for (int k = len; k < n_z; ++k) {
                const P pq = prod[(k - len) * (m >> 1) + (j >> 1)];
                siga = A::add(siga, pq.x);
                sigb = A::add(sigb, pq.y);
            }
        } else {
            siga = sigb = T(0);
        }
    }
    if (stage != nullptr) {  // fused reduction stage 1: the CTA's 512 columns are a tree node
        __syncthreads();
        T* red = prof + 4 * n_z;
        red[2 * tid] = siga;
        red[2 * tid + 1] = sigb;
        __syncthreads();
        if (threadIdx.y == 0)
            pair_node_sums<T, 2 * NT>(red, stage, nleaves, il, m);
        return;
    }
    *reinterpret_cast<P*>(part + static_cast<long long>(il) * m + j) = P{siga, sigb};
}

// K2 for fp32 with four adjacent columns per thread (m a multiple of 4): every
// stream moves as one 16-byte quad, so the fp32 sweep issues one cp.async per
// 16 bytes like the fp64 pair kernel (k_fused_spmv_pair2), and every stencil
// input — p, q, u, z(k+1), the i+-1 rows and z(j-1), z(j+4) — goes through a
// D-level cp.async ring (the fp32 pair kernel loads the neighbour rows one
// level ahead into registers, which leaves their L2 latency exposed).
// CTA = one i-plane x 1024 j. Columns j+1..j+3's south and j..j+2's north
// neighbours are lanes of the quad; the arithmetic and association are those
// of the other K2 kernels (bit-identical).
struct alignas(16) Quad {
    float x, y, z, w;
};

__device__ __forceinline__ void cpa_quad(Quad* sdst, const float* gsrc) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
}

template <bool Fast, int D, int MINB>
__global__ void __launch_bounds__(32 * kStencilWarps, MINB)
    k_fused_spmv_quad(const SlabView<float> v, float* __restrict__ u, float* __restrict__ p,
                      float* __restrict__ q, const float* __restrict__ z,
                      float* __restrict__ part, const Scalars<float>* __restrict__ S,
                      float* __restrict__ stage, int nleaves) {
    using T = float;
    using A = Ar<T, Fast>;
    constexpr int NT = 32 * kStencilWarps, NS = D + 1, CW = 4 * NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* prof = reinterpret_cast<T*>(smem_raw);
    const int n_z = v.n_z, m = v.m;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    load_profile(prof, v.prof, 4 * n_z, tid, NT);  // static data: before the dependency wait
    __syncthreads();
    pdl_wait();
    if (ld_dep(&S->done)) return;  // block-uniform
    int il = v.plane_begin + blockIdx.y;
    if (v.halo.on) {  // fused halo: boundary planes last, after the neighbours' K1 put them
        const int y = blockIdx.y, ml = v.m_loc;
        if (ml >= 3) il = y < ml - 2 ? y + 1 : (y == ml - 2 ? 0 : ml - 1);
        if (il == 0 && v.halo.ghost[0] != nullptr) halo_acquire(v.halo.wait_flag[0], v.halo.seq);
        if (il == ml - 1 && v.halo.ghost[1] != nullptr) halo_acquire(v.halo.wait_flag[1], v.halo.seq);
    }
    const int jr = blockIdx.x * CW + 4 * tid;
    const bool valid = jr < m;  // m % 4 == 0: all four columns exist
    if (stage == nullptr && !valid) return;
    const int j = valid ? jr : m - 4;
    // profile 4 n_z floats, then the ring [slot][7][NT] quads (16-byte aligned)
    Quad* ring = reinterpret_cast<Quad*>(prof + ((4 * n_z + 3) & ~3)) + tid;
    const T* sP = prof + kProfS * n_z;
    const T* bP = prof + kProfB * n_z;
    const T* cP = prof + kProfC * n_z;
    const T* dP = prof + kProfD * n_z;
    T sig[4] = {T(0), T(0), T(0), T(0)};
    if (valid) {  // the idle warps of a narrow panel's CTA (fused reduction) skip the sweep
        Col<T> cc[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) cc[t] = load_col(v, il, j + t);
        const T alpha = ld_dep(&S->alpha), beta = ld_dep(&S->beta);
        const long long base = static_cast<long long>(il) * v.plane + j;
        const T* zc = z + base;
        T* uc = u + base;
        T* pc = p + base;
        T* qc = q + base;
        const long long sm = m;
        long long oe = cc[0].oe, ow = cc[0].ow;  // same for all four columns (same plane)
        if (v.halo.on) {  // ghost rows straight from this rank's mailbox
            if (il == 0 && v.halo.ghost[0] != nullptr) ow = (v.halo.ghost[0] + j) - zc;
            if (il == v.m_loc - 1 && v.halo.ghost[1] != nullptr) oe = (v.halo.ghost[1] + j) - zc;
        }
        auto issue = [&](int k, int s) {
            const long long l = static_cast<long long>(k) * sm;
            Quad* r0 = ring + s * 7 * NT;
            cpa_quad(r0, pc + l);
            cpa_quad(r0 + NT, qc + l);
            cpa_quad(r0 + 2 * NT, uc + l);
            if (k + 1 < n_z) cpa_quad(r0 + 3 * NT, zc + l + sm);
            cpa_quad(r0 + 4 * NT, zc + l + oe);
            cpa_quad(r0 + 5 * NT, zc + l + ow);
            T* e = reinterpret_cast<T*>(r0 + 6 * NT);  // z(j-1), z(j+4) (own values on the edges)
            cpa(e, zc + l + cc[0].os);
            cpa(e + 1, zc + l + 3 + cc[3].on);
        };
#pragma unroll
        for (int t = 0; t < D; ++t) {
            if (t < n_z) issue(t, t);
            cp_commit();
        }
        Quad z0 = *reinterpret_cast<const Quad*>(zc), zd = z0;
        int cs = 0, ps_ = D;
        for (int k = 0; k < n_z; ++k) {
            const long long l = static_cast<long long>(k) * sm;
            cp_wait<D - 1>();
            const Quad* r0 = ring + cs * 7 * NT;
            const Quad pq = r0[0], qq = r0[NT], uq = r0[2 * NT];
            const Quad zu = k + 1 < n_z ? r0[3 * NT] : z0;
            const Quad ce = r0[4 * NT], cw = r0[5 * NT];
            const T* ex = reinterpret_cast<const T*>(r0 + 6 * NT);
            const T zs0 = ex[0], zn3 = ex[1];
            if (k + D < n_z) issue(k + D, ps_);
            cp_commit();
            cs = cs + 1 == NS ? 0 : cs + 1;
            ps_ = ps_ + 1 == NS ? 0 : ps_ + 1;
            const T P0[4] = {pq.x, pq.y, pq.z, pq.w}, Q0[4] = {qq.x, qq.y, qq.z, qq.w};
            const T U0[4] = {uq.x, uq.y, uq.z, uq.w}, Z0[4] = {z0.x, z0.y, z0.z, z0.w};
            const T ZU[4] = {zu.x, zu.y, zu.z, zu.w}, ZD[4] = {zd.x, zd.y, zd.z, zd.w};
            const T ZE[4] = {ce.x, ce.y, ce.z, ce.w}, ZW[4] = {cw.x, cw.y, cw.z, cw.w};
            T un[4], pn[4], qn[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                un[t] = A::add(U0[t], A::mul(alpha, P0[t]));
                pn[t] = A::add(A::mul(beta, P0[t]), Z0[t]);
                const T qb = A::mul(beta, Q0[t]);
                const T zn = t < 3 ? Z0[t + 1] : zn3;  // north: the next lane, z(j+4) at the end
                const T zs = t > 0 ? Z0[t - 1] : zs0;  // south: the previous lane, z(j-1) first
                const Col<T>& c = cc[t];
                const T dq = stencil<T, Fast>(sP[k], c.area, c.adiag, bP[k], cP[k], c.ae, c.aw,
                                              c.an, c.as, Z0[t], ZU[t], ZD[t], ZE[t], ZW[t], zn, zs);
                qn[t] = A::add(qb, A::mul(dP[k], dq));
                sig[t] = A::add(sig[t], A::mul(pn[t], qn[t]));
            }
            __stcs(reinterpret_cast<float4*>(uc + l), make_float4(un[0], un[1], un[2], un[3]));
            __stcs(reinterpret_cast<float4*>(pc + l), make_float4(pn[0], pn[1], pn[2], pn[3]));
            __stcs(reinterpret_cast<float4*>(qc + l), make_float4(qn[0], qn[1], qn[2], qn[3]));
            zd = z0;
            z0 = zu;
        }
        cp_wait<0>();
    }
    if (stage != nullptr) {  // fused reduction stage 1 (quad_node_sums)
        __syncthreads();
        T* red = prof + ((4 * n_z + 3) & ~3);
#pragma unroll
        for (int t = 0; t < 4; ++t) red[4 * tid + t] = sig[t];
        __syncthreads();
        if (threadIdx.y == 0) {
            if (m >= CW) {
                cta_subtree_sums<T, CW>(red, 1, stage, nleaves,
                                        (static_cast<long long>(il) * m + blockIdx.x * CW) / CW);
            } else {
                switch (m) {  // narrower power-of-two panel: the node is the whole plane
                    case 512: cta_subtree_sums<T, 512>(red, 1, stage, nleaves, il); break;
                    case 256: cta_subtree_sums<T, 256>(red, 1, stage, nleaves, il); break;
                    case 128: cta_subtree_sums<T, 128>(red, 1, stage, nleaves, il); break;
                    default: cta_subtree_sums<T, 64>(red, 1, stage, nleaves, il); break;
                }
            }
        }
        return;
    }
    *reinterpret_cast<float4*>(part + static_cast<long long>(il) * m + j) =
        make_float4(sig[0], sig[1], sig[2], sig[3]);
}
