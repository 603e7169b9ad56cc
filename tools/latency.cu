// Microbenchmark: dependent-chain latency (cycles/op) of DADD, DFMA, FADD, SHFL+DADD on one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double a) {
  double x = a, y = a * 0.5;
  float f = (float)a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) f = __fadd_rn(f, 1.0f);
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = __dadd_rn(z, __shfl_sync(0xffffffffu, y, i & 31));
  long long t3 = clock64();
  double m = a;
  for (int i = 0; i < n; ++i) m = __dmul_rn(m, 1.0000001);
  long long t4 = clock64();
  out[threadIdx.x] = x + f + z + m;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMallocManaged(&c, 64);
  const int n = 1 << 16;
  k<<<1, 32>>>(o, c, n, 1.0);
  cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, n, 1.0);
  cudaDeviceSynchronize();
  printf("cycles/op: dadd %.2f fadd %.2f shfl+dadd %.2f dmul %.2f\n", (double)c[0] / n, (double)c[1] / n, (double)c[2] / n, (double)c[3] / n);
  return 0;
}
