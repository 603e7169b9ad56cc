// Microbenchmark of k_eval_fold's per-cell work (K = 256, lane = 8 topics):
// rows from shared memory, dots, warp reduction, reciprocal, axpy -- how many
// SM cycles per fold cell each stage costs with 8 / 16 warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fold_micro tools/fold_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NJ = 4, KP = 256, ROWS = 96;

__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = __fma_rn(-x, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-x, r, 1.0);
  return __fma_rn(r, e, r);
}

// MODE bit 0: butterfly; bit 1: reciprocal; bit 2: axpy.  G cells per step.
template <int MODE, int G>
__global__ void k(double* out, long long* cyc, int iters) {
  extern __shared__ double rows[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x / 32;
  for (int i = tid; i < ROWS * KP; i += blockDim.x) rows[i] = 1.0 + 1e-3 * (i % 97);
  double2 th[NJ], acc[NJ];
  for (int j = 0; j < NJ; ++j) {
    th[j] = make_double2(1.0 / 256, 1.0 / 256);
    acc[j] = make_double2(0, 0);
  }
  __syncthreads();
  long long t0 = clock64();
  int f = wid * G;
  for (int it = 0; it < iters; ++it) {
    double2 r[G][NJ];
    double v[G];
#pragma unroll
    for (int c = 0; c < G; ++c) {
      const double* row = rows + ((f + c) % ROWS) * KP;
      double a = 0, b = 0;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        r[c][j] = *reinterpret_cast<const double2*>(row + 64 * j + 2 * lane);
        a = __fma_rn(th[j].x, r[c][j].x, a);
        b = __fma_rn(th[j].y, r[c][j].y, b);
      }
      v[c] = a + b;
    }
    if (MODE & 1) {
#pragma unroll
      for (int c = 0; c < G; ++c)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], o);
    }
#pragma unroll
    for (int c = 0; c < G; ++c) {
      const double s = (MODE & 2) ? rcp64(v[c]) : v[c] * 1e-3;
      if (MODE & 4) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          acc[j].x = __fma_rn(s, r[c][j].x, acc[j].x);
          acc[j].y = __fma_rn(s, r[c][j].y, acc[j].y);
        }
      } else {
        acc[0].x += s;
      }
    }
    f += nw * G;
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < NJ; ++j) s += acc[j].x + acc[j].y;
  out[blockIdx.x * blockDim.x + tid] = s;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, int G>
void run(const char* name, double* o, long long* c, int threads) {
  const int iters = 2048;
  const size_t sm = ROWS * KP * sizeof(double);
  cudaFuncSetAttribute(k<MODE, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<MODE, G><<<148, threads, sm>>>(o, c, iters);
  cudaDeviceSynchronize();
  k<MODE, G><<<148, threads, sm>>>(o, c, iters);
  cudaDeviceSynchronize();
  const double cells = double(threads / 32) * iters * G;
  printf("%-28s G=%d warps=%2d: %6.2f SM cycles per cell\n", name, G, threads / 32, double(c[0]) / cells);
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 148 * 1024 * sizeof(double));
  cudaMallocManaged(&c, 148 * sizeof(long long));
  for (int t : {256, 512}) {
    run<0, 1>("lds+dot", o, c, t);
    run<1, 1>("lds+dot+tree", o, c, t);
    run<3, 1>("lds+dot+tree+rcp", o, c, t);
    run<7, 1>("full (tree+rcp+axpy)", o, c, t);
    run<7, 2>("full (tree+rcp+axpy)", o, c, t);
    run<4, 1>("lds+dot+axpy (no tree)", o, c, t);
  }
  return 0;
}
