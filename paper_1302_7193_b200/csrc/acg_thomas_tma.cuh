// K1 / K4, TMEM-resident Thomas sweeps fed by TMA (included by acg_kernels.cu
// after acg_thomas_tm.cuh). Opt-in (ACG_THOMAS_TMA=1): measured at C3 it is
// as fast as k_thomas_tm under the power cap and 2% slower at full clock
// (K1 0.817 vs 0.799 ms), so the cp.async-ring kernel stays the default.
//
//   k_thomas_tma<Fused=true>   interleaved_prec_kernel  operator.hpp:272-346 (Alg. 3)
//   k_thomas_tma<Fused=false>  precondition             operator.hpp:141-191
//
// Same arithmetic, TMEM z', checkpointed phi and exact-recompute groups as
// k_thomas_tm; what changes is how the streamed fields reach shared memory.
// In k_thomas_tm every thread issues one cp.async per field per level plus its
// commit/wait and 64-bit address increments (~10 instructions per level, and
// the sweep is issue- and power-limited). Here the CTA (one i-plane x 128 j)
// reads each field as 2D tiles of 8 levels x 128 columns (8 KiB, fp64) with
// one cp.async.bulk.tensor per field per group, issued by a single thread into
// a ring of NSLOT group slots; completion is an mbarrier transaction count,
// slot reuse an mbarrier with one arrival per warp. The forward sweep streams
// r and q; the back substitution streams r* (written by the forward sweep,
// published to the async proxy by fence.proxy.async + a CTA barrier).
template <int CP_, int NSLOT_>
struct ThomasTmaCfg {
    static_assert(8 % CP_ == 0, "checkpoint stride divides the group of 8 levels");
    static_assert(NSLOT_ >= 2 && NSLOT_ <= 4, "2..4 group slots");
    static constexpr int W = 4, CP = CP_, NSLOT = NSLOT_, NT = 128, G = 8;
};

template <typename T, class C>
__host__ __device__ constexpr size_t thomas_tma_smem_bytes(int n_z) {
    return sizeof(T) * (static_cast<size_t>(C::NSLOT) * 2 * C::G * C::NT +
                        static_cast<size_t>(kTmProf) * n_z +
                        static_cast<size_t>((n_z + C::CP - 1) / C::CP) * C::NT);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// 2D tile (c0 = column, c1 = row) of `map` into shared memory, completing on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// Forward elimination over one group of 8 levels whose r (or y) and q warp
// tiles are in shared memory (a0 = tile0[32 t], a1 = tile1[32 t], the lane's
// column offset already applied). Full: all 8 levels exist.
template <typename T, bool Fast, bool Fused, class C, bool First, bool Full>
__device__ __forceinline__ void tma_fwd_group(const TmCol<T>& c, const T* __restrict__ prof4,
                                              int n_z, int kg, const T* tile0, const T* tile1,
                                              long long sm, T*& r_st, bool valid, TmFwd<T>& s,
                                              T* phs, T (&zb)[8]) {
    using A = Ar<T, Fast>;
    constexpr int NT = C::NT, CP = C::CP;
    const T* pg = prof4 + kg * kTmProf;
    const TmFwd<T> s0 = s;
    T nums[8];
    bool ok = true;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int k = kg + t;
        if (!Full) zb[t] = T(0);
        if (Full || k < n_z) {
            const T a0 = tile0[t * 32];
            T num = a0;
            if (Fused) {
                const T a1 = tile1[t * 32];
                s.rs = A::sub(a0, A::mul(c.alpha, a1));  // r* = r - alpha q (operator.hpp:311)
                s.r2 = A::add(s.r2, A::mul(s.rs, s.rs));
                num = s.rs;
                if (valid) *r_st = s.rs;
                r_st += sm;
            }
            nums[t] = num;
            if (First && t == 0)
                tm_level<T, Fast, Fused, true>(c, num, pg, s, ok);
            else
                tm_level<T, Fast, Fused, false>(c, num, pg + t * kTmProf, s, ok);
            zb[t] = s.zp;
            if (t % CP == 0) phs[(k / CP) * NT] = s.phi;
        }
    }
    if (!Fast && !ok) {  // rare: redo the group with the reference's divisions
        TmFwd<T> e = s0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int k = kg + t;
            if (Full || k < n_z) {
                if (First && t == 0)
                    tm_level_exact<T, Fused, true>(c, nums[t], pg, e);
                else
                    tm_level_exact<T, Fused, false>(c, nums[t], pg + t * kTmProf, e);
                zb[t] = e.zp;
                if (t % CP == 0) phs[(k / CP) * NT] = e.phi;
            }
        }
        s.phi = e.phi;
        s.zp = e.zp;
    }
}

// Back substitution over one group (levels kg+7 .. kg, those above `top`
// skipped unless Full); r* of the group in the warp tile tile0[32 t].
template <typename T, bool Fast, bool Fused, class C, bool Full>
__device__ __forceinline__ void tma_bwd_group(const TmCol<T>& c, const T* __restrict__ prof4,
                                              int top, int kg, unsigned tma_addr, const T* phs,
                                              const T* tile0, long long sm, T*& z_st, bool valid,
                                              T& zn, T& kap) {
    using A = Ar<T, Fast>;
    constexpr int NT = C::NT, CP = C::CP;
    T zq[8];
    tm_ld8(tma_addr, zq);
    const T* pg = prof4 + kg * kTmProf;
    T ph[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int k = kg + t;
        const T* pk = pg + t * kTmProf;
        if (!Full && k > top)
            ph[t] = T(0);
        else if (t % CP == 0)
            ph[t] = phs[(k / CP) * NT];
        else if (Fast)
            ph[t] = pk[1] * fast_rcp(pivot_k<T, Fast>(pk[0], c.at, pk[2], ph[t - 1]));
        else  // phi is data-independent: its range was validated per context
            ph[t] = div_fast(pk[1], pivot_k<T, Fast>(pk[0], c.at, pk[2], ph[t - 1]));
    }
#pragma unroll
    for (int t = 7; t >= 0; --t) {
        const int k = kg + t;
        if (!Full && k > top) continue;
        const T zs = A::sub(zq[t], A::mul(ph[t], zn));
        if (Fused) kap = A::add(kap, A::mul(zs, tile0[t * 32]));
        if (valid) __stcs(z_st, zs);
        z_st -= sm;
        zn = zs;
    }
}

// Rows of the 2D view of a field: row (il + 1) * n_z + k holds level k of
// plane il (row 0.. n_z-1 is the ghost plane before the slab). Each warp owns
// its 32 columns' tiles (box 32 x 8 levels) and its own ring of NSLOT group
// slots with one full-barrier each; lane 0 is the warp's producer, so warps
// never wait for each other.
template <typename T, bool Fast, bool Fused, class C>
__global__ void __launch_bounds__(C::NT)
    k_thomas_tma(const SlabView<T> v, const __grid_constant__ CUtensorMap map0,
                 const __grid_constant__ CUtensorMap map1, T* __restrict__ r,
                 const T* __restrict__ in, T* __restrict__ out, T* __restrict__ part_r2,
                 T* __restrict__ part_k, const Scalars<T>* __restrict__ S,
                 const Scalars<T>* __restrict__ gate, unsigned tcols, T* __restrict__ stage,
                 int nleaves) {
    using A = Ar<T, Fast>;
    constexpr int NT = C::NT, NSLOT = C::NSLOT, G = C::G, W = C::W;
    constexpr int NARR = Fused ? 2 : 1;
    constexpr int WT = G * 32;  // values of one warp tile (8 levels x 32 columns)
    constexpr unsigned kTileBytes = WT * sizeof(T);
    constexpr unsigned kColsPer8 = 8u * sizeof(T) / 4u;
    if (Fused ? S->done != 0 : (gate != nullptr && gate->done != 0)) return;  // block-uniform
    __shared__ unsigned tm_slot;
    __shared__ __align__(8) unsigned long long full[W][NSLOT];
    extern __shared__ __align__(1024) unsigned char smem_tma[];
    T* ring_all = reinterpret_cast<T*>(smem_tma);  // TMA destinations need 128 B alignment
    T* prof4 = ring_all + NSLOT * 2 * G * NT;
    const int n_z = v.n_z, m = v.m;
    const int warp = threadIdx.y;
    const int lane = threadIdx.x;
    const int tid = warp * 32 + lane;
    T* ring = ring_all + warp * NSLOT * 2 * WT;  // this warp's [slot][array][8][32]
    unsigned long long* fb = full[warp];
    const int il = blockIdx.y;
    const int j0 = blockIdx.x * NT;
    const int jw = j0 + warp * 32;
    const int row0 = (il + 1) * n_z;  // row of level 0 of this plane in the 2D view
    const int ngf = (n_z + G - 1) / G;  // forward groups
    const int top = n_z - 2;
    const int ngb = Fused && top >= 0 ? top / G + 1 : 0;  // backward groups (r* re-read)
    if (warp == 0) tm_alloc(&tm_slot, tcols);
    if (tid == 0 && (smem_u32(ring_all) & 127u) != 0) __trap();
    if (lane == 0) {
        for (int q = 0; q < NSLOT; ++q) mbar_init(&fb[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // sequence number q: forward groups 0..ngf-1, then backward groups ngf..;
    // slot q % NSLOT, phase (q / NSLOT) & 1. Producer: lane 0 of the warp.
    auto issue = [&](int q) {
        const int sl = q % NSLOT;
        T* dst = ring + sl * 2 * WT;
        if (q < ngf) {
            mbar_expect_tx(&fb[sl], NARR * kTileBytes);
            tma_load_2d(dst, &map0, jw, row0 + q * G, &fb[sl]);
            if (Fused) tma_load_2d(dst + WT, &map1, jw, row0 + q * G, &fb[sl]);
        } else {
            const int kg = (top / G - (q - ngf)) * G;
            mbar_expect_tx(&fb[sl], kTileBytes);
            tma_load_2d(dst, &map0, jw, row0 + kg, &fb[sl]);
        }
    };
    __syncwarp();
    if (lane == 0)
        for (int q = 0; q < NSLOT && q < ngf; ++q) issue(q);
    for (int e = tid; e < kTmProf * n_z; e += NT) {
        const int k = e / kTmProf, row = e % kTmProf;
        const int src = row < 3 ? row : (Fast ? kProfInvD : kProfD);
        prof4[e] = v.prof[src * n_z + k];
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();

    const unsigned tm = tm_slot + (static_cast<unsigned>(32 * warp) << 16);
    const int jr = jw + lane;
    const bool valid = jr < m;
    const int j = valid ? jr : m - 1;
    T* phs = prof4 + kTmProf * n_z + tid;  // [checkpoint][NT]
    const long long ncol = static_cast<long long>(v.m_loc) * m;
    const long long cidx = static_cast<long long>(il) * m + j;
    TmCol<T> c;
    c.area = v.col[kColArea * ncol + cidx];
    c.at = v.col[kColAtil * ncol + cidx];
    c.inva = v.col[kColInvA * ncol + cidx];
    c.alpha = Fused ? S->alpha : T(0);
    const long long base = static_cast<long long>(il) * v.plane + j;
    T* const rc = Fused ? r + base : nullptr;
    T* const oc = out + base;
    const long long sm = m;
    (void)in;

    // ------------------------------------------------------------ forward
    T* r_st = rc;
    TmFwd<T> s{T(0), T(0), T(0), T(0)};
    for (int g = 0; g < ngf; ++g) {
        const int sl = g % NSLOT;
        mbar_wait(&fb[sl], (g / NSLOT) & 1);
        const T* t0 = ring + sl * 2 * WT + lane;
        const T* t1 = t0 + WT;
        T zb[8];
        const int kg = g * G;
        if (g == 0) {
            if (n_z >= 8)
                tma_fwd_group<T, Fast, Fused, C, true, true>(c, prof4, n_z, 0, t0, t1, sm, r_st,
                                                             valid, s, phs, zb);
            else
                tma_fwd_group<T, Fast, Fused, C, true, false>(c, prof4, n_z, 0, t0, t1, sm, r_st,
                                                              valid, s, phs, zb);
        } else if (kg + 8 <= n_z) {
            tma_fwd_group<T, Fast, Fused, C, false, true>(c, prof4, n_z, kg, t0, t1, sm, r_st,
                                                          valid, s, phs, zb);
        } else {
            tma_fwd_group<T, Fast, Fused, C, false, false>(c, prof4, n_z, kg, t0, t1, sm, r_st,
                                                           valid, s, phs, zb);
        }
        tm_st8(tm + static_cast<unsigned>(g) * kColsPer8, zb);
        __syncwarp();  // every lane has read the slot
        const int qn = g + NSLOT;
        if (lane == 0 && qn < ngf) issue(qn);
    }
    tm_wait_st();
    if (valid) oc[static_cast<long long>(n_z - 1) * sm] = s.zp;

    // ------------------------------------------------------------ backward
    // z_{n-1} = z'_{n-1}; z_k = z'_k - phi_k z_{k+1}; kappa from the top (:329-335)
    if (Fused) {
        // this warp's r* stores -> visible to its TMA (async proxy) re-reads
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
        if (lane == 0)
            for (int q = ngf; q < ngf + NSLOT && q < ngf + ngb; ++q) issue(q);
    }
    T kap = Fused ? A::mul(s.zp, s.rs) : T(0);
    T zn = s.zp;
    T* z_st = oc + static_cast<long long>(top) * sm;
    for (int b = 0; b < (top >= 0 ? top / G + 1 : 0); ++b) {
        const int kg = (top / G - b) * G;
        const int q = ngf + b;
        const T* t0 = nullptr;
        if (Fused) {
            const int sl = q % NSLOT;
            mbar_wait(&fb[sl], (q / NSLOT) & 1);
            t0 = ring + sl * 2 * WT + lane;
        }
        const unsigned ta = tm + static_cast<unsigned>(kg / G) * kColsPer8;
        if (kg + 7 > top)
            tma_bwd_group<T, Fast, Fused, C, false>(c, prof4, top, kg, ta, phs, t0, sm, z_st,
                                                    valid, zn, kap);
        else
            tma_bwd_group<T, Fast, Fused, C, true>(c, prof4, top, kg, ta, phs, t0, sm, z_st,
                                                   valid, zn, kap);
        if (Fused) {
            __syncwarp();
            if (lane == 0 && q + NSLOT < ngf + ngb) issue(q + NSLOT);
        }
    }
    if (Fused && stage == nullptr && valid) {
        part_r2[cidx] = s.r2;
        part_k[cidx] = kap;
    }
    if (Fused && stage != nullptr) {  // fused reduction stage 1 (one plane x 128 j)
        __syncthreads();
        T* red = ring_all;  // every TMA tile has been consumed
        red[tid] = s.r2;
        red[NT + tid] = kap;
        __syncthreads();
        if (warp == 0)
            cta_subtree_sums<T, NT>(red, 2, stage, nleaves,
                                    (static_cast<long long>(il) * m + j0) / NT);
    }
    tm_fence_before();
    __syncthreads();
    if (warp == 0) {
        tm_fence_after();
        tm_dealloc(tm_slot, tcols);
    }
}
