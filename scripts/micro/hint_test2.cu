// Policy variants: evict_last / evict_normal / runtime select (diagnostic microtest)
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long pl() { unsigned long long p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ unsigned long long pn() { unsigned long long p; asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ unsigned long long pfst() { unsigned long long p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ void st(double* o, double v, unsigned long long p) { asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(o), "d"(v), "l"(p) : "memory"); }
__global__ void k_last(double* o, unsigned long long* u) { u[threadIdx.x] = pl(); st(o + threadIdx.x, 1.0, pl()); }
__global__ void k_normal(double* o, unsigned long long* u) { u[threadIdx.x] = pn(); st(o + threadIdx.x, 1.0, pn()); }
__global__ void k_select(double* o, int h) { unsigned long long p = h ? pfst() : pn(); st(o + threadIdx.x, 1.0, p); }
__global__ void k_select2(double* o, int h) { unsigned long long p = h ? pl() : pfst(); st(o + threadIdx.x, 1.0, p); }
int main() {
  double* o; unsigned long long* u; cudaMalloc(&o, 4096); cudaMalloc(&u, 4096);
  for (int t = 0; t < 6; ++t) {
    switch (t) { case 0: k_last<<<1,32>>>(o, u); break; case 1: k_normal<<<1,32>>>(o, u); break;
      case 2: k_select<<<1,32>>>(o, 1); break; case 3: k_select<<<1,32>>>(o, 0); break;
      case 4: k_select2<<<1,32>>>(o, 1); break; case 5: k_select2<<<1,32>>>(o, 0); break; }
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0; cudaMemcpy(&h, u, 8, cudaMemcpyDeviceToHost);
    printf("case %d: %s policy=0x%llx\n", t, cudaGetErrorString(e), h);
    if (e != cudaSuccess) { cudaDeviceReset(); cudaMalloc(&o, 4096); cudaMalloc(&u, 4096); }
  }
}
