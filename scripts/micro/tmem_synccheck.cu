// Minimal tcgen05 kernel for the compute-sanitizer synccheck question
// (tests/test_sanitizers.py): does synccheck accept a CTA that only
// allocates, relinquishes and frees tensor memory, with the documented
// fences and one __syncthreads? If it reports "Barrier error ... Missing
// init" here, the report on k_thomas_tm is the tool's, not the kernel's.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tmem_synccheck tmem_synccheck.cu
#include <cstdio>

__global__ void k_tmem_alloc_only(unsigned* out) {
    __shared__ unsigned taddr;
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&taddr));
    const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(sa)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned t = taddr;
    if (threadIdx.x == 0) out[blockIdx.x] = t;
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t) : "memory");
}

int main() {
    unsigned* d = nullptr;
    cudaMalloc(&d, 4 * sizeof(unsigned));
    k_tmem_alloc_only<<<4, 128>>>(d);
    const cudaError_t e = cudaDeviceSynchronize();
    unsigned h[4] = {0, 0, 0, 0};
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    std::printf("tmem_synccheck: %s, taddr %u %u %u %u\n", cudaGetErrorString(e), h[0], h[1], h[2],
                h[3]);
    return e == cudaSuccess ? 0 : 1;
}
