// Streaming roofline for the read/write mixes of the PCG sweeps: copy (1R:1W),
// K1-like (2R:2W: r R+W, q R, z W) and K2-like (4R:3W: u,p,q R+W, z R), fp64,
// 1.07 GB per field (C3), double2 vector accesses, CUDA-event timed.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_22(double2* __restrict__ r, const double2* __restrict__ q, double2* __restrict__ z, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double2 a = r[i], b = q[i]; a.x -= 0.5 * b.x; a.y -= 0.5 * b.y; r[i] = a; z[i] = make_double2(a.x * 3, a.y * 3);
  }
}
__global__ void k_43(double2* __restrict__ u, double2* __restrict__ p, double2* __restrict__ q, const double2* __restrict__ z, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double2 pu = p[i], qu = q[i], uu = u[i], zz = z[i];
    uu.x += 0.3 * pu.x; uu.y += 0.3 * pu.y; pu.x = zz.x + 0.2 * pu.x; pu.y = zz.y + 0.2 * pu.y;
    qu.x = zz.x + 0.2 * qu.x; qu.y = zz.y + 0.2 * qu.y; u[i] = uu; p[i] = pu; q[i] = qu;
  }
}
int main() {
  const long N = 1024L * 1024 * 128, n = N / 2;
  double2 *a, *b, *c, *d;
  cudaMalloc(&a, N * 8); cudaMalloc(&b, N * 8); cudaMalloc(&c, N * 8); cudaMalloc(&d, N * 8);
  cudaMemset(a, 0, N * 8); cudaMemset(b, 0, N * 8); cudaMemset(c, 0, N * 8); cudaMemset(d, 0, N * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int g : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) for (int bs : {256, 512}) {
    float best[3] = {1e9, 1e9, 1e9};
    for (int rep = 0; rep < 6; ++rep) {
      float ms;
      cudaEventRecord(e0); k_copy<<<g, bs>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (ms < best[0]) best[0] = ms;
      cudaEventRecord(e0); k_22<<<g, bs>>>(a, b, c, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (ms < best[1]) best[1] = ms;
      cudaEventRecord(e0); k_43<<<g, bs>>>(a, b, c, d, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (ms < best[2]) best[2] = ms;
    }
    printf("grid %5d block %3d  copy %7.1f GB/s  2R2W(K1) %7.1f GB/s  4R3W(K2) %7.1f GB/s\n", g, bs,
           2.0 * N * 8 / best[0] / 1e6, 4.0 * N * 8 / best[1] / 1e6, 7.0 * N * 8 / best[2] / 1e6);
  }
  return 0;
}
