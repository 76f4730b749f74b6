// K1 / K4: per-column Thomas sweeps (included by acg_kernels.cu).
//
//   k_thomas<Fused=true>   interleaved_prec_kernel  operator.hpp:272-346 (paper Alg. 3)
//   k_thomas<Fused=false>  precondition             operator.hpp:141-191
//
// One thread owns one column; a warp is 32 consecutive j of one i-plane, so
// every level is one coalesced row per field.
//
// Memory pipeline. The forward elimination streams r and q (K1) or y (K4) up
// the column through a per-thread shared-memory ring filled by cp.async
// (LDGSTS) D levels ahead: the copies are asynchronous, so D*16 B per thread
// stay in flight without tying up registers. r* and z' go straight to their
// output fields; the back substitution streams them back, most recent first,
// through the same ring while they are still L2-resident (the DRAM traffic of
// the sweep stays at the 4 algorithmic references per point).
//
// phi_k = b'_k / D_k is needed again by the back substitution. Storing it for
// every level (n_z*s bytes per column) is what limits the columns in flight,
// so only every CP-th phi is kept in shared memory and the others are
// recomputed during the back substitution with the identical operation
// sequence (same bits), off the z critical path.
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

// One forward-elimination step of the pivot recurrence (operator.hpp:318-321):
//   D_k = ((a'_k - b'_k - c'_k) - alpha~) - phi_{k-1} c'_k,   phi_k = b'_k / D_k
template <typename T, bool Fast>
__device__ __forceinline__ T pivot(int k, T sk, T at, T ck, T phi_prev) {
    using A = Ar<T, Fast>;
    return k == 0 ? A::sub(sk, at) : A::sub(A::sub(sk, at), A::mul(phi_prev, ck));
}
template <typename T, bool Fast>
__device__ __forceinline__ T phi_of(T bk, T D) {
    if (Fast) return bk * (T(1) / D);
    return Ar<T, false>::div(bk, D);
}

template <int W_, int CP_, int D_>
struct ThomasCfg {
    static constexpr int W = W_, CP = CP_, D = D_, NT = 32 * W_, NS = D_ + 1;
};

template <typename T, class C>
__host__ __device__ constexpr size_t thomas_smem_bytes(int n_z, bool global_phi) {
    return sizeof(T) * (static_cast<size_t>(kProfRows) * n_z +
                        (global_phi ? 0 : static_cast<size_t>((n_z + C::CP - 1) / C::CP) * C::NT) +
                        static_cast<size_t>(C::NS) * 2 * C::NT);
}

template <typename T, bool Fast, bool Fused, class C>
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

    T* phs = prof + kProfRows * n_z;
    T* ring = phs + (phi_g ? 0 : static_cast<size_t>((n_z + CP - 1) / CP) * NT);
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
    T* rc = Fused ? r + base : nullptr;
    const T* ic = in + base;
    T* oc = out + base;
    // phi checkpoint c (level c*CP): shared [c][tid] or global plane-major rows
    auto phi_slot = [&](int c) -> T* {
        return phi_g ? phi_g + base + static_cast<long long>(c) * m : phs + c * NT + tid;
    };
    auto slot = [&](int s, int a) -> T* { return ring + (s * 2 + a) * NT + tid; };

    // ------------------------------------------------------------ forward
#pragma unroll
    for (int t = 0; t < D; ++t) {
        if (t < n_z) {
            const long long l = static_cast<long long>(t) * m;
            if (Fused) {
                cpa(slot(t, 0), rc + l);
                cpa(slot(t, 1), ic + l);
            } else {
                cpa(slot(t, 0), ic + l);
            }
        }
        cp_commit();
    }
    int cs = 0, ps = D;
    T r2 = T(0), phi = T(0), zp = T(0), rs = T(0);
    bool bad = false;
    for (int k = 0; k < n_z; ++k) {
        cp_wait<D - 1>();
        const T a0 = *slot(cs, 0);
        const T a1 = Fused ? *slot(cs, 1) : T(0);
        const int kn = k + D;
        if (kn < n_z) {
            const long long l = static_cast<long long>(kn) * m;
            if (Fused) {
                cpa(slot(ps, 0), rc + l);
                cpa(slot(ps, 1), ic + l);
            } else {
                cpa(slot(ps, 0), ic + l);
            }
        }
        cp_commit();
        cs = cs + 1 == NS ? 0 : cs + 1;
        ps = ps + 1 == NS ? 0 : ps + 1;

        T num = a0;
        if (Fused) {
            rs = A::sub(a0, A::mul(alpha, a1));  // r* = r - alpha q (operator.hpp:311)
            r2 = A::add(r2, A::mul(rs, rs));
            num = rs;
        }
        const T Dk = pivot<T, Fast>(k, sP[k], at, cP[k], phi);
        bad |= (Dk == T(0));
        if (Fast) {
            const T rD = T(1) / Dk;
            phi = bP[k] * rD;
            zp = (k == 0) ? num * (inva * idP[0]) * rD : (num * (inva * idP[k]) - cP[k] * zp) * rD;
        } else {
            phi = A::div(bP[k], Dk);
            if (Fused)  // z'_0 = r*/(D_0 |T| d_0) (:312), z'_k (:321-324)
                zp = (k == 0) ? A::div(num, A::mul(A::mul(Dk, area), dP[0]))
                              : A::div(A::sub(A::div(num, A::mul(area, dP[k])), A::mul(cP[k], zp)), Dk);
            else        // x'_0 = y/(|T| d_0)/D_0 (:174), x'_k (:183)
                zp = (k == 0) ? A::div(A::div(num, A::mul(area, dP[0])), Dk)
                              : A::div(A::sub(A::div(num, A::mul(area, dP[k])), A::mul(cP[k], zp)), Dk);
        }
        const long long l = static_cast<long long>(k) * m;
        if (Fused) rc[l] = rs;
        oc[l] = zp;
        if (k % CP == 0) *phi_slot(k / CP) = phi;
    }
    if (bad) {
        S->pivot = 1;
        return;
    }
    // ------------------------------------------------------------ backward
    // z_{n-1} = z'_{n-1}; z_k = z'_k - phi_k z_{k+1}; kappa from the top (:329-335)
    cp_wait<0>();
    __threadfence_block();  // own z', r* stores before the async re-reads
    T kap = Fused ? A::mul(zp, rs) : T(0);
    T zn = zp;
    int issue = n_z - 2;
#pragma unroll
    for (int t = 0; t < D; ++t) {
        if (issue >= 0) {
            const long long l = static_cast<long long>(issue) * m;
            cpa(slot(t, 0), oc + l);
            if (Fused) cpa(slot(t, 1), rc + l);
            --issue;
        }
        cp_commit();
    }
    cs = 0;
    ps = D;
    int top = n_z - 2;
    int seg0 = top >= 0 ? (top / CP) * CP : -1;
    while (seg0 >= 0) {
        T ph[CP];
        ph[0] = *phi_slot(seg0 / CP);
#pragma unroll
        for (int t = 1; t < CP; ++t) {
            const int kk = seg0 + t;
            ph[t] = ph[t - 1];
            if (kk <= top) ph[t] = phi_of<T, Fast>(bP[kk], pivot<T, Fast>(kk, sP[kk], at, cP[kk], ph[t - 1]));
        }
#pragma unroll
        for (int t = CP - 1; t >= 0; --t) {
            const int kk = seg0 + t;
            if (kk <= top) {
                cp_wait<D - 1>();
                const T zk = *slot(cs, 0);
                const T rk = Fused ? *slot(cs, 1) : T(0);
                if (issue >= 0) {
                    const long long l = static_cast<long long>(issue) * m;
                    cpa(slot(ps, 0), oc + l);
                    if (Fused) cpa(slot(ps, 1), rc + l);
                    --issue;
                }
                cp_commit();
                cs = cs + 1 == NS ? 0 : cs + 1;
                ps = ps + 1 == NS ? 0 : ps + 1;
                const T zs = A::sub(zk, A::mul(ph[t], zn));
                if (Fused) kap = A::add(kap, A::mul(zs, rk));
                __stcs(oc + static_cast<long long>(kk) * m, zs);
                zn = zs;
            }
        }
        top = seg0 - 1;
        seg0 -= CP;
    }
    cp_wait<0>();
    if (Fused) {
        part_r2[cidx] = r2;
        part_k[cidx] = kap;
    }
}
