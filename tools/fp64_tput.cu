// Microbenchmark: per-SM throughput of DFMA (independent chains), f64 SHFL
// and LDS.128 on this B200, and DFMA dependent-chain latency -- the numbers
// that size the held-out evaluation kernel (k_eval_fold).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_tput tools/fp64_tput.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_dfma(double* out, long long* cyc, int n) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = 1.0 + threadIdx.x * 1e-9 + c * 1e-7;
  const double a = 0.999999, b = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __fma_rn(x[c], a, b);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_shfl(double* out, long long* cyc, int n) {
  double x[4] = {1.0 * threadIdx.x, 2.0, 3.0, 4.0};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = __shfl_xor_sync(0xffffffffu, x[c], (i + c) & 31);
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x[0] + x[1] + x[2] + x[3];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_lds(double* out, long long* cyc, int n) {
  extern __shared__ double2 sm2[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm2[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  const int lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double2 v = sm2[((i * 8 + c) * 32 + lane) & 4095];
      acc.x += v.x;
      acc.y += v.y;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 148 * 1024 * sizeof(double));
  cudaMallocManaged(&c, 148 * sizeof(long long));
  const int n = 4096;
  for (int threads : {32, 256, 512, 1024}) {
    k_dfma<8><<<148, threads>>>(o, c, n);
    cudaDeviceSynchronize();
    k_dfma<8><<<148, threads>>>(o, c, n);
    cudaDeviceSynchronize();
    const double ops = double(threads) * n * 8;  // per SM (one block per SM)
    printf("DFMA  %4d threads/SM: %.1f lane-ops/clk/SM\n", threads, ops / double(c[0]));
  }
  k_dfma<1><<<1, 32>>>(o, c, n);
  cudaDeviceSynchronize();
  k_dfma<1><<<1, 32>>>(o, c, n);
  cudaDeviceSynchronize();
  printf("DFMA dependent latency: %.2f clk\n", double(c[0]) / n);
  for (int threads : {256, 1024}) {
    k_shfl<<<148, threads>>>(o, c, n);
    cudaDeviceSynchronize();
    k_shfl<<<148, threads>>>(o, c, n);
    cudaDeviceSynchronize();
    printf("SHFL.f64 %4d threads/SM: %.2f warp-shfl(f64)/clk/SM\n", threads,
           double(threads / 32) * n * 4 / double(c[0]));
  }
  for (int threads : {256, 1024}) {
    k_lds<<<148, threads, 65536>>>(o, c, n);
    cudaDeviceSynchronize();
    k_lds<<<148, threads, 65536>>>(o, c, n);
    cudaDeviceSynchronize();
    printf("LDS.128 %4d threads/SM: %.1f B/clk/SM\n", threads,
           double(threads) * n * 8 * 16 / double(c[0]));
  }
  return 0;
}
