// K1 / K4, TMEM-resident Thomas sweeps with two columns per thread (included
// by acg_kernels.cu after acg_thomas_tm.cuh). Opt-in (ACG_THOMAS_TM2=1): with
// one warp per scheduler the second recurrence does not hide the FP64 chain
// latency that the second warp of k_thomas_tm hides (C3: 0.99 vs 0.80 ms), so
// it is kept as a measured alternative, not the default.
//
//   k_thomas_tm2<Fused=true>   interleaved_prec_kernel  operator.hpp:272-346 (Alg. 3)
//   k_thomas_tm2<Fused=false>  precondition             operator.hpp:141-191
//
// Why two columns per thread. TMEM holds z' for 256 fp64 columns of 128 levels
// per SM; k_thomas_tm spends them on 256 threads (8 warps, one column each) and
// is issue-bound (~92 instructions per column-level, issue active ~48%): all
// the streaming bookkeeping (cp.async, ring waits, 64-bit address updates,
// profile loads, TMEM transfers, loop control) is paid per column. Here 128
// threads (one persistent 4-warp CTA per SM) each own two adjacent columns:
// every load, store and ring operation moves the pair as one 16-byte vector,
// the profile loads are shared, and the two independent recurrences give each
// warp the instruction-level parallelism the halved warp count takes away.
// Arithmetic, exact-recompute groups and TMEM staging are those of k_thomas_tm
// (bit-identical results).
template <int CP_, int D_, int DB_>
struct ThomasTm2Cfg {
    static_assert(D_ >= 1 && D_ <= 15 && DB_ >= 1 && DB_ <= 15, "prefetch depth below the ring size");
    static_assert(8 % CP_ == 0, "checkpoint stride divides the group of 8 levels");
    static constexpr int W = 4, CP = CP_, D = D_, DB = DB_, NT = 128, NS = 16, COLS = 2 * NT;
};

template <typename T>
struct alignas(2 * sizeof(T)) Pair {
    T x, y;
};

template <typename T, class C>
__host__ __device__ constexpr size_t thomas_tm2_smem_bytes(int n_z) {
    return sizeof(T) * (static_cast<size_t>(kTmProf) * n_z +
                        2 * static_cast<size_t>((n_z + C::CP - 1) / C::CP) * C::NT +
                        static_cast<size_t>(C::NS) * 2 * 2 * C::NT);
}

// 16- (fp64) or 8-byte (fp32) pair load through L2 (ld.global.cg).
template <typename T>
__device__ __forceinline__ Pair<T> ldcg_pair(const T* p) {
    if constexpr (sizeof(T) == 8) {
        const double2 d = __ldcg(reinterpret_cast<const double2*>(p));
        return Pair<T>{d.x, d.y};
    } else {
        const float2 f = __ldcg(reinterpret_cast<const float2*>(p));
        return Pair<T>{f.x, f.y};
    }
}

template <typename T>
__device__ __forceinline__ void cpa_pair(Pair<T>* sdst, const T* gsrc) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
    if constexpr (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}

// Ring slot (16 slots) of level kg + o for a group base kg (multiple of 8).
template <typename T>
__device__ __forceinline__ Pair<T>* ring2_at(Pair<T>* cur, Pair<T>* oth, int o, int NT) {
    return (o >= 0 && o < 8) ? cur + (2 * o) * NT
         : (o >= 8 && o < 16) ? oth + (2 * (o - 8)) * NT
         : (o >= 16) ? cur + (2 * (o - 16)) * NT
         : (o >= -8) ? oth + (2 * (o + 8)) * NT
                     : cur + (2 * (o + 16)) * NT;
}

// Forward elimination of both columns over one group of 8 levels.
template <typename T, bool Fast, bool Fused, class C, bool First, bool Full>
__device__ __forceinline__ void tm2_fwd_group(const TmCol<T>& ca, const TmCol<T>& cb,
                                              const T* __restrict__ prof4, int n_z, int kg,
                                              Pair<T>* cur, Pair<T>* oth, const T*& ia_n,
                                              const T*& ib_n, long long sm, T*& r_st, bool valid,
                                              TmFwd<T>& sa, TmFwd<T>& sb, T* phs,
                                              T (&za)[8], T (&zb)[8]) {
    using A = Ar<T, Fast>;
    constexpr int NT = C::NT, D = C::D, CP = C::CP;
    const T* pg = prof4 + kg * kTmProf;
    const TmFwd<T> sa0 = sa, sb0 = sb;
    T na[8], nb[8];
    bool ok = true;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int k = kg + t;
        if (!Full) {
            za[t] = T(0);
            zb[t] = T(0);
        }
        if (Full || k < n_z) {
            cp_wait<D - 1>();
            const Pair<T> a0 = cur[(2 * t) * NT];
            const Pair<T> a1 = Fused ? cur[(2 * t + 1) * NT] : Pair<T>{T(0), T(0)};
            if (k + D < n_z) {
                Pair<T>* dst = ring2_at<T>(cur, oth, t + D, NT);
                cpa_pair<T>(dst, ia_n);
                if (Fused) cpa_pair<T>(dst + NT, ib_n);
            }
            cp_commit();
            ia_n += sm;
            ib_n += sm;
            T numa = a0.x, numb = a0.y;
            if (Fused) {
                sa.rs = A::sub(a0.x, A::mul(ca.alpha, a1.x));  // r* = r - alpha q (operator.hpp:311)
                sb.rs = A::sub(a0.y, A::mul(cb.alpha, a1.y));
                sa.r2 = A::add(sa.r2, A::mul(sa.rs, sa.rs));
                sb.r2 = A::add(sb.r2, A::mul(sb.rs, sb.rs));
                numa = sa.rs;
                numb = sb.rs;
                if (valid) *reinterpret_cast<Pair<T>*>(r_st) = Pair<T>{sa.rs, sb.rs};
                r_st += sm;
            }
            na[t] = numa;
            nb[t] = numb;
            if (First && t == 0) {
                tm_level<T, Fast, Fused, true>(ca, numa, pg, sa, ok);
                tm_level<T, Fast, Fused, true>(cb, numb, pg, sb, ok);
            } else {
                tm_level<T, Fast, Fused, false>(ca, numa, pg + t * kTmProf, sa, ok);
                tm_level<T, Fast, Fused, false>(cb, numb, pg + t * kTmProf, sb, ok);
            }
            za[t] = sa.zp;
            zb[t] = sb.zp;
            if (t % CP == 0) {
                phs[(2 * (k / CP)) * NT] = sa.phi;
                phs[(2 * (k / CP) + 1) * NT] = sb.phi;
            }
        }
    }
    if (!Fast && !ok) {  // rare: redo the group with the reference's divisions
        TmFwd<T> ea = sa0, eb = sb0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int k = kg + t;
            if (Full || k < n_z) {
                if (First && t == 0) {
                    tm_level_exact<T, Fused, true>(ca, na[t], pg, ea);
                    tm_level_exact<T, Fused, true>(cb, nb[t], pg, eb);
                } else {
                    tm_level_exact<T, Fused, false>(ca, na[t], pg + t * kTmProf, ea);
                    tm_level_exact<T, Fused, false>(cb, nb[t], pg + t * kTmProf, eb);
                }
                za[t] = ea.zp;
                zb[t] = eb.zp;
                if (t % CP == 0) {
                    phs[(2 * (k / CP)) * NT] = ea.phi;
                    phs[(2 * (k / CP) + 1) * NT] = eb.phi;
                }
            }
        }
        sa.phi = ea.phi;
        sa.zp = ea.zp;
        sb.phi = eb.phi;
        sb.zp = eb.zp;
    }
}

// Back substitution of both columns over one group (levels kg+7 .. kg).
template <typename T, bool Fast, bool Fused, class C, bool Full>
__device__ __forceinline__ void tm2_bwd_group(const TmCol<T>& ca, const TmCol<T>& cb,
                                              const T* __restrict__ prof4, int top, int kg,
                                              unsigned ta, unsigned tb, const T* phs,
                                              Pair<T>* cur, Pair<T>* oth, const T*& ra_n,
                                              long long sm, T*& z_st, bool valid, T& zna,
                                              T& znb, T& kapa, T& kapb) {
    using A = Ar<T, Fast>;
    constexpr int NT = C::NT, D = C::DB, CP = C::CP;
    T qa[8], qb[8];
    tm_ld8(ta, qa);
    tm_ld8(tb, qb);
    const T* pg = prof4 + kg * kTmProf;
    T pa[8], pb[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int k = kg + t;
        const T* pk = pg + t * kTmProf;
        if (!Full && k > top) {
            pa[t] = T(0);
            pb[t] = T(0);
        } else if (t % CP == 0) {
            pa[t] = phs[(2 * (k / CP)) * NT];
            pb[t] = phs[(2 * (k / CP) + 1) * NT];
        } else if (Fast) {
            pa[t] = pk[1] * fast_rcp(pivot_k<T, Fast>(pk[0], ca.at, pk[2], pa[t - 1]));
            pb[t] = pk[1] * fast_rcp(pivot_k<T, Fast>(pk[0], cb.at, pk[2], pb[t - 1]));
        } else {  // data-independent phi: its range was validated per context
            pa[t] = div_fast(pk[1], pivot_k<T, Fast>(pk[0], ca.at, pk[2], pa[t - 1]));
            pb[t] = div_fast(pk[1], pivot_k<T, Fast>(pk[0], cb.at, pk[2], pb[t - 1]));
        }
    }
#pragma unroll
    for (int t = 7; t >= 0; --t) {
        const int k = kg + t;
        if (!Full && k > top) continue;
        Pair<T> rk{T(0), T(0)};
        if (Fused) {
            cp_wait<D - 1>();
            rk = cur[(2 * t) * NT];
            if (k - D >= 0) cpa_pair<T>(ring2_at<T>(cur, oth, t - D, NT), ra_n);
            cp_commit();
            ra_n -= sm;
        }
        const T za = A::sub(qa[t], A::mul(pa[t], zna));
        const T zb = A::sub(qb[t], A::mul(pb[t], znb));
        if (Fused) {
            kapa = A::add(kapa, A::mul(za, rk.x));
            kapb = A::add(kapb, A::mul(zb, rk.y));
        }
        if (valid) {
            if constexpr (sizeof(T) == 8)
                __stcs(reinterpret_cast<double2*>(z_st), make_double2(za, zb));
            else
                __stcs(reinterpret_cast<float2*>(z_st), make_float2(za, zb));
        }
        z_st -= sm;
        zna = za;
        znb = zb;
    }
}

// Persistent: grid <= #SMs, one 4-warp CTA per SM owning all 512 TMEM columns;
// tile = one i-plane x 256 j (thread tid: columns j0 + 2 tid, + 1).
template <typename T, bool Fast, bool Fused, class C>
__global__ void __launch_bounds__(C::NT, 1)
    k_thomas_tm2(const SlabView<T> v, T* __restrict__ r, const T* __restrict__ in,
                 T* __restrict__ out, T* __restrict__ part_r2, T* __restrict__ part_k,
                 const Scalars<T>* __restrict__ S, const Scalars<T>* __restrict__ gate,
                 unsigned tcols, T* __restrict__ stage, int nleaves, int ntiles, int tiles_row) {
    using A = Ar<T, Fast>;
    constexpr int NT = C::NT, D = C::D, CP = C::CP;
    constexpr unsigned kColsPer8 = 8u * sizeof(T) / 4u;
    if (Fused ? S->done != 0 : (gate != nullptr && gate->done != 0)) return;  // grid-uniform
    __shared__ unsigned tm_slot;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* prof4 = reinterpret_cast<T*>(smem_raw);
    const int n_z = v.n_z, m = v.m;
    const int warp = threadIdx.y;
    const int tid = warp * 32 + threadIdx.x;
    if (warp == 0) tm_alloc(&tm_slot, tcols);
    for (int e = tid; e < kTmProf * n_z; e += NT) {
        const int k = e / kTmProf, row = e % kTmProf;
        const int src = row < 3 ? row : (Fast ? kProfInvD : kProfD);
        prof4[e] = v.prof[src * n_z + k];
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const int nck = (n_z + CP - 1) / CP;
    T* phs = prof4 + kTmProf * n_z + tid;  // [checkpoint][2][NT]
    Pair<T>* ring = reinterpret_cast<Pair<T>*>(prof4 + kTmProf * n_z + 2 * nck * NT) + tid;  // [16][2][NT]
    const unsigned tma = tm_slot + (static_cast<unsigned>(32 * warp) << 16);
    const unsigned tmb = tma + tcols / 2;
    const long long ncol = static_cast<long long>(v.m_loc) * m;
    const long long sm = m;
    const int top = n_z - 2;

    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int il = tile / tiles_row;
        if (v.halo.on && il > 0)  // fused halo: the boundary planes first, their z travels
            il = il == 1 ? v.m_loc - 1 : il - 1;
        const int j0 = (tile % tiles_row) * C::COLS;
        const int jr = j0 + 2 * tid;
        const bool valid = jr < m;  // m even: both columns of the pair exist
        const int j = valid ? jr : m - 2;
        const long long cia = static_cast<long long>(il) * m + j;
        TmCol<T> ca, cb;
        ca.area = v.col[kColArea * ncol + cia];
        cb.area = v.col[kColArea * ncol + cia + 1];
        ca.at = v.col[kColAtil * ncol + cia];
        cb.at = v.col[kColAtil * ncol + cia + 1];
        ca.inva = v.col[kColInvA * ncol + cia];
        cb.inva = v.col[kColInvA * ncol + cia + 1];
        ca.alpha = cb.alpha = Fused ? S->alpha : T(0);
        const long long base = static_cast<long long>(il) * v.plane + j;
        T* const rc = Fused ? r + base : nullptr;
        const T* const ic = in + base;
        T* const oc = out + base;

        // -------------------------------------------------------- forward
        const T* ia_n = Fused ? rc : ic;
        const T* ib_n = ic;
#pragma unroll
        for (int t = 0; t < D; ++t) {
            if (t < n_z) {
                cpa_pair<T>(ring + (2 * t) * NT, ia_n);
                if (Fused) cpa_pair<T>(ring + (2 * t + 1) * NT, ib_n);
            }
            cp_commit();
            ia_n += sm;
            ib_n += sm;
        }
        T* r_st = rc;
        TmFwd<T> sa{T(0), T(0), T(0), T(0)}, sb{T(0), T(0), T(0), T(0)};
        {
            T za[8], zb[8];
            if (n_z >= 8)
                tm2_fwd_group<T, Fast, Fused, C, true, true>(ca, cb, prof4, n_z, 0, ring,
                                                             ring + 16 * NT, ia_n, ib_n, sm, r_st,
                                                             valid, sa, sb, phs, za, zb);
            else
                tm2_fwd_group<T, Fast, Fused, C, true, false>(ca, cb, prof4, n_z, 0, ring,
                                                              ring + 16 * NT, ia_n, ib_n, sm, r_st,
                                                              valid, sa, sb, phs, za, zb);
            tm_st8(tma, za);
            tm_st8(tmb, zb);
        }
        int kg = 8;
        for (; kg + 8 <= n_z; kg += 8) {
            T za[8], zb[8];
            Pair<T>* cur = ring + (kg & 8) * 2 * NT;
            Pair<T>* oth = ring + ((kg + 8) & 8) * 2 * NT;
            tm2_fwd_group<T, Fast, Fused, C, false, true>(ca, cb, prof4, n_z, kg, cur, oth, ia_n,
                                                          ib_n, sm, r_st, valid, sa, sb, phs, za,
                                                          zb);
            const unsigned off = static_cast<unsigned>(kg / 8) * kColsPer8;
            tm_st8(tma + off, za);
            tm_st8(tmb + off, zb);
        }
        if (kg < n_z) {
            T za[8], zb[8];
            Pair<T>* cur = ring + (kg & 8) * 2 * NT;
            Pair<T>* oth = ring + ((kg + 8) & 8) * 2 * NT;
            tm2_fwd_group<T, Fast, Fused, C, false, false>(ca, cb, prof4, n_z, kg, cur, oth,
                                                           ia_n, ib_n, sm, r_st, valid, sa, sb,
                                                           phs, za, zb);
            const unsigned off = static_cast<unsigned>(kg / 8) * kColsPer8;
            tm_st8(tma + off, za);
            tm_st8(tmb + off, zb);
        }
        tm_wait_st();
        cp_wait<0>();

        // -------------------------------------------------------- backward
        __threadfence_block();  // own r* stores before the async re-reads
        if (valid)
            *reinterpret_cast<Pair<T>*>(oc + static_cast<long long>(n_z - 1) * sm) =
                Pair<T>{sa.zp, sb.zp};
        T kapa = Fused ? A::mul(sa.zp, sa.rs) : T(0);
        T kapb = Fused ? A::mul(sb.zp, sb.rs) : T(0);
        T zna = sa.zp, znb = sb.zp;
        const T* ra_n = nullptr;
        if (Fused) {
            const T* ra = rc + static_cast<long long>(top) * sm;
            for (int t = 0; t < C::DB; ++t) {
                const int k = top - t;
                if (k >= 0) cpa_pair<T>(ring + (2 * (k & 15)) * NT, ra);
                cp_commit();
                ra -= sm;
            }
            ra_n = rc + static_cast<long long>(top - C::DB) * sm;
        }
        T* z_st = oc + static_cast<long long>(top) * sm;
        if (top >= 0) {
            int g = (top / 8) * 8;
            if (g + 7 > top) {
                const unsigned off = static_cast<unsigned>(g / 8) * kColsPer8;
                tm2_bwd_group<T, Fast, Fused, C, false>(
                    ca, cb, prof4, top, g, tma + off, tmb + off, phs, ring + (g & 8) * 2 * NT,
                    ring + ((g + 8) & 8) * 2 * NT, ra_n, sm, z_st, valid, zna, znb, kapa, kapb);
                g -= 8;
            }
            for (; g >= 0; g -= 8) {
                const unsigned off = static_cast<unsigned>(g / 8) * kColsPer8;
                tm2_bwd_group<T, Fast, Fused, C, true>(
                    ca, cb, prof4, top, g, tma + off, tmb + off, phs, ring + (g & 8) * 2 * NT,
                    ring + ((g + 8) & 8) * 2 * NT, ra_n, sm, z_st, valid, zna, znb, kapa, kapb);
            }
        }
        cp_wait<0>();
        if (v.halo.on) {  // fused halo: z columns of a boundary plane -> neighbour's mailbox
#pragma unroll
            for (int sd = 0; sd < 2; ++sd) {
                if (v.halo.put[sd] == nullptr || il != (sd == 0 ? 0 : v.m_loc - 1)) continue;
                if (valid) {
                    T* dst = v.halo.put[sd] + j;
                    for (int k0 = 0; k0 < n_z; k0 += 8) {
                        Pair<T> t8[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (k0 + u < n_z)
                                t8[u] = ldcg_pair<T>(oc + static_cast<long long>(k0 + u) * sm);
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (k0 + u < n_z)
                                *reinterpret_cast<Pair<T>*>(dst + static_cast<long long>(k0 + u) * sm) =
                                    t8[u];
                    }
                    __threadfence_system();
                }
                __syncthreads();  // tile-uniform branch
                if (tid == 0) {
                    __threadfence_system();
                    if (atomicAdd(v.halo.arrive + sd, 1u) == static_cast<unsigned>(tiles_row) - 1) {
                        atomicExch(v.halo.arrive + sd, 0u);
                        __threadfence_system();
                        st_release_sys(v.halo.put_flag[sd], v.halo.seq);
                    }
                }
            }
        }
        if (Fused && stage == nullptr && valid) {
            *reinterpret_cast<Pair<T>*>(part_r2 + cia) = Pair<T>{sa.r2, sb.r2};
            *reinterpret_cast<Pair<T>*>(part_k + cia) = Pair<T>{kapa, kapb};
        }
        if (Fused && stage != nullptr) {  // fused reduction stage 1: the tile is a tree node
            T* red = reinterpret_cast<T*>(ring - tid);  // ring drained (cp_wait<0>) by everyone
            __syncthreads();
            red[2 * tid] = sa.r2;
            red[2 * tid + 1] = sb.r2;
            red[2 * NT + 2 * tid] = kapa;
            red[2 * NT + 2 * tid + 1] = kapb;
            __syncthreads();
            if (warp < 2)
                cta_subtree_sums<T, 2 * NT>(red + warp * 2 * NT, 1, stage + warp * nleaves,
                                            nleaves, (static_cast<long long>(il) * m + j0) / (2 * NT));
            __syncthreads();
        }
    }
    tm_fence_before();
    __syncthreads();
    if (warp == 0) {
        tm_fence_after();
        tm_dealloc(tm_slot, tcols);
    }
}
