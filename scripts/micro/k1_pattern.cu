// K1's memory pattern without its arithmetic: how fast can the exact sweep's
// traffic go at the occupancy the real kernel has? C3 (1024^2 x 128 fp64,
// plane-major [il][k][j]): one thread per column, CTA = one plane x 128 j,
// 4 planes per CTA; forward reads r, q through a 16-slot cp.async ring 15
// levels ahead and writes r* = r - alpha q; backward re-reads r* top-down
// through the ring (L2) and writes z = r* + 0.5 z_{k+1}. Dynamic shared
// memory is padded to hold `ctas` CTAs per SM (k_thomas_tm: 2, by TMEM).
// Prints ms per launch (CUDA events, 20 launches after 3 warm-up) and the
// algorithmic 4.31 GB model rate.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o k1_pattern k1_pattern.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

constexpr int NZ = 128, NT = 128, NS = 16, D = 15;
__constant__ int cM, cTPC;  // panel width, planes per CTA (argv)

__device__ __forceinline__ void cpa8(double* s, const double* g) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void wait_g() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// DEFER: the z stores of plane p move into the forward sweep of plane p + 1
// (k_thomas_tm would read them back from TMEM), so both phases mix reads and
// writes; the CTA's last plane flushes its z after its backward sweep.
// TOPREG: the backward sweep takes the top 16 levels' r* from registers (kept
// from the end of the forward sweep) and re-reads only the levels below.
// PREF: the next plane's first D levels (r into a side buffer, q into the
// ring's q slots, which the backward sweep does not use) are issued when the
// backward sweep starts, so the next forward sweep starts with a full ring.
template <bool DEFER, bool TOPREG = false, bool PREF = false>
__global__ void __launch_bounds__(NT) k_pattern(double* __restrict__ r, const double* __restrict__ q,
                                                 double* __restrict__ z, double alpha) {
    extern __shared__ double ring_all[];  // [slot][2][NT], then (PREF) [D][NT]
    const int tid = threadIdx.x;
    double* ring = ring_all + tid;
    double* side = ring_all + NS * 2 * NT + tid;
    bool prefetched = false;
    const int M = cM, TPC = cTPC;
    const long long plane = static_cast<long long>(NZ) * M;
    for (int rep = 0; rep < TPC; ++rep) {
        const int il = blockIdx.y * TPC + rep;
        if (il >= static_cast<int>(gridDim.y) * TPC || il >= M) break;
        const int j = blockIdx.x * NT + tid;
        double* rc = r + il * plane + j;
        const double* qc = q + il * plane + j;
        double* zc = z + il * plane + j;
        if (PREF && prefetched) {
            wait_g<0>();
            for (int t = 0; t < D; ++t) ring[(2 * t) * NT] = side[t * NT];
            for (int t = 0; t < D; ++t) commit();  // keep the group count of the prefill
        } else {
            for (int t = 0; t < D; ++t) {
                cpa8(ring + (2 * t) * NT, rc + static_cast<long long>(t) * M);
                cpa8(ring + (2 * t + 1) * NT, qc + static_cast<long long>(t) * M);
                commit();
            }
        }
        prefetched = false;
        double top = 0.0;
        double keep[16];
        double* zprev = z + (il - 1) * plane + j;  // DEFER: the previous plane's z
        for (int k = 0; k < NZ; ++k) {
            wait_g<D - 1>();
            const double rv = ring[(2 * (k % NS)) * NT], qv = ring[(2 * (k % NS) + 1) * NT];
            if (k + D < NZ) {
                cpa8(ring + (2 * ((k + D) % NS)) * NT, rc + static_cast<long long>(k + D) * M);
                cpa8(ring + (2 * ((k + D) % NS) + 1) * NT, qc + static_cast<long long>(k + D) * M);
            }
            commit();
            const double rs = rv - alpha * qv;
            rc[static_cast<long long>(k) * M] = rs;
            if (DEFER && rep > 0) zprev[static_cast<long long>(k) * M] = rs * 0.25;
            if (TOPREG && k >= NZ - 16) keep[k - (NZ - 16)] = rs;
            top = rs;
        }
        wait_g<0>();
        __threadfence_block();
        if (PREF && rep + 1 < TPC && il + 1 < M) {  // next plane's first levels
            const double* rn = r + (il + 1) * plane + j;
            const double* qn = q + (il + 1) * plane + j;
            for (int t = 0; t < D; ++t) {
                cpa8(side + t * NT, rn + static_cast<long long>(t) * M);
                cpa8(ring + (2 * t + 1) * NT, qn + static_cast<long long>(t) * M);
            }
            commit();
            prefetched = true;
        }
        const int kb = TOPREG ? NZ - 17 : NZ - 2;  // first level re-read from memory
        for (int t = 0; t < D; ++t) {
            const int k = kb - t;
            if (k >= 0) cpa8(ring + (2 * (k % NS)) * NT, rc + static_cast<long long>(k) * M);
            commit();
        }
        double zn = top;
        if (!DEFER || rep == TPC - 1) zc[static_cast<long long>(NZ - 1) * M] = zn;
        if (TOPREG) {
#pragma unroll
            for (int k = NZ - 2; k > NZ - 17; --k) {
                zn = keep[k - (NZ - 16)] + 0.5 * zn;
                if (!DEFER || rep == TPC - 1) zc[static_cast<long long>(k) * M] = zn;
            }
        }
        for (int k = kb; k >= 0; --k) {
            wait_g<D - 1>();
            const double rk = ring[(2 * (k % NS)) * NT];
            if (k - D >= 0) cpa8(ring + (2 * ((k - D) % NS)) * NT, rc + static_cast<long long>(k - D) * M);
            commit();
            zn = rk + 0.5 * zn;
            if (!DEFER || rep == TPC - 1) zc[static_cast<long long>(k) * M] = zn;
        }
        wait_g<0>();
        __syncthreads();
    }
}

int main(int argc, char** argv) {
    const int M = argc > 1 ? std::atoi(argv[1]) : 1024, TPC = argc > 2 ? std::atoi(argv[2]) : 4;
    cudaMemcpyToSymbol(cM, &M, sizeof(int));
    cudaMemcpyToSymbol(cTPC, &TPC, sizeof(int));
    std::printf("m = %d, n_z = %d, %d planes per CTA\n", M, NZ, TPC);
    const size_t n = static_cast<size_t>(M) * M * NZ;
    double *r, *q, *z;
    cudaMalloc(&r, n * 8);
    cudaMalloc(&q, n * 8);
    cudaMalloc(&z, n * 8);
    cudaMemset(r, 0, n * 8);
    cudaMemset(q, 0, n * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const dim3 grid(M / NT, (M + TPC - 1) / TPC), block(NT);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int defer = 0; defer < 4; ++defer)
    for (int ctas : {2, 3, 4}) {
        auto kern = defer == 3 ? k_pattern<false, false, true>
                  : defer == 2 ? k_pattern<false, true> : defer ? k_pattern<true> : k_pattern<false>;
        size_t smem = 233472 / (ctas + 1) - 1024 + 64;  // the k_thomas_tm padding rule
        const size_t ring = static_cast<size_t>(NS) * 2 * NT * 8 + (defer == 3 ? D * NT * 8 : 0);
        if (smem < ring) smem = ring;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
        for (int i = 0; i < 3; ++i) kern<<<grid, block, smem>>>(r, q, z, 0.37);
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) kern<<<grid, block, smem>>>(r, q, z, 0.37);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 20;
        const double model = 4.0 * n * 8 + 2.0 * M * M * 8;  // K1's algorithmic bytes
        std::printf("%s CTAs/SM %d (occupancy %d, %d warps/SM): %.3f ms per launch = %.0f GB/s of the model\n",
                    defer == 3 ? "prefetch:  " : defer == 2 ? "top r* reg:" : defer ? "deferred z:" : "as K1:     ", ctas, occ, occ * 4, ms, model / ms / 1e6);
    }
    std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
