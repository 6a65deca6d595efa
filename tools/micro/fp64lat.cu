// Single-warp dependent-chain latency (cycles per op) of the FP64 building
// blocks the scorer's critical path is made of: DADD, DMUL, DFMA, dmax
// (DSETP + FSEL), rsqrt.approx.ftz.f64 (MUFU.RSQ64H), the branch-free
// correctly rounded sqrt, and a shared-memory load (LDS.64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64lat.cu -o fp64lat
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double sqrt_fast(double s) {
  double y0;
  asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(s));
  const double e = __fma_rn(-s, __dmul_rn(y0, y0), 1.0);
  const double y1 = __fma_rn(__fma_rn(e, 0.375, 0.5), __dmul_rn(y0, e), y0);
  const double q = __dmul_rn(s, y1);
  const double d = __fma_rn(-q, q, s);
  return __fma_rn(d, __dmul_rn(y1, 0.5), q);
}

template <int OP>
__global__ void lat(int iters, double a, double* sink, long long* cyc) {
  __shared__ double sh[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sh[i] = 0.0;
  __syncthreads();
  double x = 1.0 + threadIdx.x * 1e-9;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) x = __dadd_rn(x, a);
    if (OP == 1) x = __dmul_rn(x, a);
    if (OP == 2) x = __fma_rn(x, a, a);
    if (OP == 3) x = x > a ? x : a + 0.0 * x;  // dmax via compare + select
    if (OP == 4) {
      double y;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
      x = y;
    }
    if (OP == 5) x = sqrt_fast(x);
    if (OP == 6) x = sh[(__double2loint(x) & 0) + (i & 31)] + x;  // LDS + DADD
    if (OP == 7) x = fmax(x, a);
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  sink[threadIdx.x] = x;
}

int main() {
  double* sink;
  long long* cyc;
  cudaMalloc(&sink, 1024 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  const char* names[] = {"DADD", "DMUL", "DFMA", "dmax(DSETP+FSEL)", "MUFU.RSQ64H", "sqrt_fast", "LDS+DADD", "fmax"};
  const int iters = 4096;
  for (int op = 0; op < 8; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: lat<0><<<1, 32>>>(iters, 1e-20, sink, cyc); break;
        case 1: lat<1><<<1, 32>>>(iters, 1.0000001, sink, cyc); break;
        case 2: lat<2><<<1, 32>>>(iters, 0.5, sink, cyc); break;
        case 3: lat<3><<<1, 32>>>(iters, 0.5, sink, cyc); break;
        case 4: lat<4><<<1, 32>>>(iters, 0.5, sink, cyc); break;
        case 5: lat<5><<<1, 32>>>(iters, 0.5, sink, cyc); break;
        case 6: lat<6><<<1, 32>>>(iters, 0.5, sink, cyc); break;
        case 7: lat<7><<<1, 32>>>(iters, 0.5, sink, cyc); break;
      }
    }
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    std::printf("%-18s %6.1f cycles/op (single warp, dependent chain)\n", names[op], double(c) / iters);
  }
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
