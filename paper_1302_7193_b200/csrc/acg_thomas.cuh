// K1 / K4: per-column Thomas sweeps (included by acg_kernels.cu).
//
//   k_thomas<Fused=true>   interleaved_prec_kernel  operator.hpp:272-346 (paper Alg. 3)
//   k_thomas<Fused=false>  precondition             operator.hpp:141-191
//
// One thread owns one column; a warp is 32 consecutive j of one i-plane, so
// every level is one coalesced row per field.
//
// Memory pipeline. The forward elimination streams r and q (K1) or y (K4) up
// the column through a per-thread 8-slot shared-memory ring filled by cp.async
// (LDGSTS) D <= 7 levels ahead: the copies are asynchronous, so D*16 B per
// thread stay in flight without tying up registers, and because the loop is
// unrolled by the ring size every slot address is a compile-time offset.
// r* and z' go straight to their output fields; the back substitution streams
// them back, most recent first, through the same ring while they are still
// L2-resident (the sweep's DRAM traffic stays near 4 references per point).
//
// phi_k = b'_k / D_k is needed again by the back substitution. Storing it for
// every level (n_z*s bytes per column) is what limits the columns in flight,
// so only every CP-th phi is kept (shared memory, or an HBM scratch field for
// very tall columns) and the others are recomputed in the back substitution
// with the identical operation sequence (same bits).
template <typename T>
__device__ __forceinline__ void cpa(T* sdst, const T* gsrc) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
    if constexpr (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Reciprocal for the FAST path: rcp.approx + two Newton steps (~1 ulp).
__device__ __forceinline__ double fast_rcp(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    e = fma(-d, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ float fast_rcp(float d) { return __frcp_rn(d); }

// One step of the pivot recurrence (operator.hpp:318-321):
//   D_k = ((a'_k - b'_k - c'_k) - alpha~) - phi_{k-1} c'_k,   phi_k = b'_k / D_k
template <typename T, bool Fast>
__device__ __forceinline__ T pivot_k(T sk, T at, T ck, T phi_prev) {
    using A = Ar<T, Fast>;
    return A::sub(A::sub(sk, at), A::mul(phi_prev, ck));
}

template <int W_, int CP_, int D_>
struct ThomasCfg {
    static_assert(D_ >= 1 && D_ <= 7, "ring of 8 slots");
    static_assert(8 % CP_ == 0, "checkpoint stride divides the unroll");
    static constexpr int W = W_, CP = CP_, D = D_, NT = 32 * W_, NS = 8;
};

template <typename T, class C>
__host__ __device__ constexpr size_t thomas_smem_bytes(int n_z, bool global_phi) {
    return sizeof(T) * (static_cast<size_t>(kProfRows) * n_z +
                        (global_phi ? 0 : static_cast<size_t>((n_z + C::CP - 1) / C::CP) * C::NT) +
                        static_cast<size_t>(C::NS) * 2 * C::NT);
}

template <typename T, bool Fast, bool Fused, class C, bool GPhi>
__global__ void __launch_bounds__(C::NT)
    k_thomas(const SlabView<T> v, T* __restrict__ r, const T* __restrict__ in,
             T* __restrict__ out, T* __restrict__ part_r2, T* __restrict__ part_k,
             Scalars<T>* __restrict__ S, const Scalars<T>* __restrict__ gate,
             T* __restrict__ phi_g) {
    using A = Ar<T, Fast>;
    constexpr int NT = C::NT, NS = C::NS, D = C::D, CP = C::CP;
    if (Fused ? S->done != 0 : (gate != nullptr && gate->done != 0)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* prof = reinterpret_cast<T*>(smem_raw);
    const int n_z = v.n_z, m = v.m;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    load_profile(prof, v.prof, kProfRows * n_z, tid, NT);
    __syncthreads();
    const int j = blockIdx.x * 32 + threadIdx.x;
    const int il = blockIdx.y * C::W + threadIdx.y;
    if (j >= m || il >= v.m_loc) return;

    const int nck = (n_z + CP - 1) / CP;
    T* phs = prof + kProfRows * n_z + tid;                  // [checkpoint][NT]
    T* ring = prof + kProfRows * n_z + (GPhi ? 0 : nck * NT) + tid;  // [slot][2][NT]
    const T* sP = prof + kProfS * n_z;
    const T* bP = prof + kProfB * n_z;
    const T* cP = prof + kProfC * n_z;
    const T* dP = prof + kProfD * n_z;
    const T* idP = prof + kProfInvD * n_z;
    const long long ncol = static_cast<long long>(v.m_loc) * m;
    const long long cidx = static_cast<long long>(il) * m + j;
    const T area = v.col[kColArea * ncol + cidx];
    const T at = v.col[kColAtil * ncol + cidx];
    const T inva = v.col[kColInvA * ncol + cidx];
    const T alpha = Fused ? S->alpha : T(0);
    const long long base = static_cast<long long>(il) * v.plane + j;
    T* const rc = Fused ? r + base : nullptr;
    const T* const ic = in + base;
    T* const oc = out + base;
    T* const pg = GPhi ? phi_g + base : nullptr;
    const long long sm = m;  // level stride

    // ------------------------------------------------------------ forward
    // slot of level k = k % 8; level k + D is issued into slot (k + D) % 8,
    // consumed at iteration k - 1 (D <= 7).
    const T* ia = Fused ? rc : ic;  // ring array 0 source
    const T* ib = ic;               // ring array 1 source (fused: q)
#pragma unroll
    for (int t = 0; t < D; ++t) {
        if (t < n_z) {
            cpa(ring + (2 * t) * NT, ia + t * sm);
            if (Fused) cpa(ring + (2 * t + 1) * NT, ib + t * sm);
        }
        cp_commit();
    }
    const T* ia_n = ia + D * sm;  // next level to issue
    const T* ib_n = ib + D * sm;
    T* r_st = rc;
    T* o_st = oc;

    T r2 = T(0), phi = T(0), zp = T(0), rs = T(0);
    bool bad = false;
    // level 0 (peeled: z'_0 = r*/((D_0 |T|) d_0), operator.hpp:312; x'_0 = y/(|T| d_0)/D_0, :174)
    {
        cp_wait<D - 1>();
        const T a0 = ring[0];
        const T a1 = Fused ? ring[NT] : T(0);
        if (D < n_z) {
            cpa(ring + (2 * D) * NT, ia_n);
            if (Fused) cpa(ring + (2 * D + 1) * NT, ib_n);
        }
        cp_commit();
        ia_n += sm;
        ib_n += sm;
        T num = a0;
        if (Fused) {
            rs = A::sub(a0, A::mul(alpha, a1));
            r2 = A::add(r2, A::mul(rs, rs));
            num = rs;
        }
        const T D0 = A::sub(sP[0], at);
        bad |= (D0 == T(0));
        if (Fast) {
            const T rD = fast_rcp(D0);
            phi = bP[0] * rD;
            zp = num * (inva * idP[0]) * rD;
        } else {
            phi = A::div(bP[0], D0);
            zp = Fused ? A::div(num, A::mul(A::mul(D0, area), dP[0]))
                       : A::div(A::div(num, A::mul(area, dP[0])), D0);
        }
        if (Fused) *r_st = rs;
        *o_st = zp;
        r_st += sm;
        o_st += sm;
        if (GPhi) pg[0] = phi; else phs[0] = phi;
    }
    for (int k0 = 0; k0 < n_z; k0 += NS) {
#pragma unroll
        for (int t = 0; t < NS; ++t) {
            const int k = k0 + t;
            if (k == 0 || k >= n_z) continue;
            cp_wait<D - 1>();
            const T a0 = ring[(2 * t) * NT];
            const T a1 = Fused ? ring[(2 * t + 1) * NT] : T(0);
            if (k + D < n_z) {
                cpa(ring + (2 * ((t + D) % NS)) * NT, ia_n);
                if (Fused) cpa(ring + (2 * ((t + D) % NS) + 1) * NT, ib_n);
            }
            cp_commit();
            ia_n += sm;
            ib_n += sm;
            T num = a0;
            if (Fused) {
                rs = A::sub(a0, A::mul(alpha, a1));  // r* = r - alpha q (operator.hpp:311)
                r2 = A::add(r2, A::mul(rs, rs));
                num = rs;
            }
            const T Dk = pivot_k<T, Fast>(sP[k], at, cP[k], phi);
            bad |= (Dk == T(0));
            if (Fast) {
                const T rD = fast_rcp(Dk);
                phi = bP[k] * rD;
                zp = (num * (inva * idP[k]) - cP[k] * zp) * rD;
            } else {  // operator.hpp:320-324 / :181-183
                phi = A::div(bP[k], Dk);
                zp = A::div(A::sub(A::div(num, A::mul(area, dP[k])), A::mul(cP[k], zp)), Dk);
            }
            if (Fused) *r_st = rs;
            *o_st = zp;
            r_st += sm;
            o_st += sm;
            if (t % CP == 0) {
                if (GPhi)
                    pg[(k / CP) * sm] = phi;
                else
                    phs[(k0 / CP + t / CP) * NT] = phi;
            }
        }
    }
    if (bad) {
        S->pivot = 1;
        cp_wait<0>();
        return;
    }
    // ------------------------------------------------------------ backward
    // z_{n-1} = z'_{n-1}; z_k = z'_k - phi_k z_{k+1}; kappa from the top (:329-335)
    cp_wait<0>();
    __threadfence_block();  // own z', r* stores before the async re-reads
    T kap = Fused ? A::mul(zp, rs) : T(0);
    T zn = zp;
    // level k uses slot k % 8; level k - D is issued into slot (k - D) % 8 = (k + 8 - D) % 8
    const int top = n_z - 2;
    {
        const T* oa = oc + static_cast<long long>(top) * sm;
        const T* ra = Fused ? rc + static_cast<long long>(top) * sm : nullptr;
#pragma unroll
        for (int t = 0; t < D; ++t) {
            const int k = top - t;
            if (k >= 0) {
                const int s = k & (NS - 1);
                cpa(ring + (2 * s) * NT, oa);
                if (Fused) cpa(ring + (2 * s + 1) * NT, ra);
            }
            cp_commit();
            oa -= sm;
            if (Fused) ra -= sm;
        }
    }
    const T* oa_n = oc + static_cast<long long>(top - D) * sm;  // next level to issue
    const T* ra_n = Fused ? rc + static_cast<long long>(top - D) * sm : nullptr;
    T* z_st = oc + static_cast<long long>(top) * sm;
    for (int k0 = (top >= 0 ? (top / NS) * NS : -NS); k0 >= 0; k0 -= NS) {
        // phi for the levels of this chunk, recomputed from the checkpoints
        T ph[NS];
#pragma unroll
        for (int t = 0; t < NS; ++t) {
            const int k = k0 + t;
            if (k > top)
                ph[t] = T(0);
            else if (t % CP == 0)
                ph[t] = GPhi ? pg[(k / CP) * sm] : phs[(k0 / CP + t / CP) * NT];
            else
                ph[t] = Fast ? bP[k] * fast_rcp(pivot_k<T, Fast>(sP[k], at, cP[k], ph[t - 1]))
                             : A::div(bP[k], pivot_k<T, Fast>(sP[k], at, cP[k], ph[t - 1]));
        }
#pragma unroll
        for (int t = NS - 1; t >= 0; --t) {
            const int k = k0 + t;
            if (k > top) continue;
            cp_wait<D - 1>();
            const T zk = ring[(2 * t) * NT];
            const T rk = Fused ? ring[(2 * t + 1) * NT] : T(0);
            if (k - D >= 0) {
                const int s = (t + NS - D) % NS;
                cpa(ring + (2 * s) * NT, oa_n);
                if (Fused) cpa(ring + (2 * s + 1) * NT, ra_n);
            }
            cp_commit();
            oa_n -= sm;
            if (Fused) ra_n -= sm;
            const T zs = A::sub(zk, A::mul(ph[t], zn));
            if (Fused) kap = A::add(kap, A::mul(zs, rk));
            __stcs(z_st, zs);
            z_st -= sm;
            zn = zs;
        }
    }
    cp_wait<0>();
    if (Fused) {
        part_r2[cidx] = r2;
        part_k[cidx] = kap;
    }
}

