// Which L2 cache-hint forms run on this B200? (diagnostic microtest)
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long pol_first() { unsigned long long p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ unsigned long long pol_first_f32() { unsigned long long p; asm volatile("createpolicy.fractional.L2::evict_first.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p)); return p; }
__global__ void k_create(unsigned long long* o) { o[threadIdx.x] = pol_first(); }
__global__ void k_ld(const double* a, double* o) {
  unsigned long long p = pol_first(); double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a + threadIdx.x), "l"(p));
  o[threadIdx.x] = v; }
__global__ void k_st(double* o) {
  unsigned long long p = pol_first();
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(o + threadIdx.x), "d"(1.0), "l"(p) : "memory"); }
__global__ void k_cpa(const double* a, double* o) {
  __shared__ double s[64];
  unsigned long long p = pol_first();
  unsigned sa = (unsigned)__cvta_generic_to_shared(s + threadIdx.x);
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" :: "r"(sa), "l"(a + threadIdx.x), "l"(p) : "memory");
  asm volatile("cp.async.commit_group;"); asm volatile("cp.async.wait_group 0;" ::: "memory");
  o[threadIdx.x] = s[threadIdx.x]; }
__global__ void k_cpa_cg(const double* a, double* o) {
  __shared__ double s[64];
  unsigned long long p = pol_first();
  unsigned sa = (unsigned)__cvta_generic_to_shared(s + 2 * (threadIdx.x / 2));
  if (threadIdx.x % 2 == 0)
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" :: "r"(sa), "l"(a + threadIdx.x), "l"(p) : "memory");
  asm volatile("cp.async.commit_group;"); asm volatile("cp.async.wait_group 0;" ::: "memory");
  o[threadIdx.x] = s[threadIdx.x]; }
__global__ void k_ldlast(const double* a, double* o) {
  double v; asm volatile("ld.global.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(a + threadIdx.x));
  o[threadIdx.x] = v; }
int main() {
  double *a, *o; unsigned long long* u;
  cudaMalloc(&a, 1024); cudaMalloc(&o, 1024); cudaMalloc(&u, 1024); cudaMemset(a, 0, 1024);
  const char* names[] = {"createpolicy", "ld.hint", "st.hint", "cp.async.ca.hint", "cp.async.cg.hint", "ld.L1::evict_last"};
  for (int t = 0; t < 6; ++t) {
    switch (t) {
      case 0: k_create<<<1, 32>>>(u); break;
      case 1: k_ld<<<1, 32>>>(a, o); break;
      case 2: k_st<<<1, 32>>>(o); break;
      case 3: k_cpa<<<1, 32>>>(a, o); break;
      case 4: k_cpa_cg<<<1, 32>>>(a, o); break;
      case 5: k_ldlast<<<1, 32>>>(a, o); break;
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%-20s %s\n", names[t], cudaGetErrorString(e));
    if (e != cudaSuccess) { cudaDeviceReset(); cudaMalloc(&a, 1024); cudaMalloc(&o, 1024); cudaMalloc(&u, 1024); cudaMemset(a, 0, 1024); }
  }
  unsigned long long h; cudaMemcpy(&h, u, 8, cudaMemcpyDeviceToHost); printf("policy=0x%llx\n", h);
}
