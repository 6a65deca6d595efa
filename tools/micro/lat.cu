// Microbenchmarks: FP64 dependent-chain latency and throughput on this device.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat_dadd(double* out, long long* cyc, int n, double a) {
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x; cyc[threadIdx.x] = t1 - t0;
}
__global__ void lat_dmul(double* out, long long* cyc, int n, double a) {
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x; cyc[threadIdx.x] = t1 - t0;
}
__global__ void lat_dfma(double* out, long long* cyc, int n, double a) {
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __fma_rn(x, a, 1e-300);
  long long t1 = clock64();
  out[threadIdx.x] = x; cyc[threadIdx.x] = t1 - t0;
}
__global__ void lat_lds(double* out, long long* cyc, int n) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = idx[j];
  long long t1 = clock64();
  out[threadIdx.x] = j; cyc[threadIdx.x] = t1 - t0;
}
__global__ void thr_dadd(double* out, int n, double a) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(x[k], a);
  double s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}
__global__ void thr_dfma(double* out, int n, double a) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __fma_rn(x[k], a, 1e-300);
  double s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}
__global__ void syncthreads_cost(long long* cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1 << 20);
  long long h;
  const int n = 4096;
  lat_dadd<<<1, 32>>>(out, cyc, n, 1e-12); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("DADD latency %.2f cyc\n", double(h) / n);
  lat_dmul<<<1, 32>>>(out, cyc, n, 1.0000001); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("DMUL latency %.2f cyc\n", double(h) / n);
  lat_dfma<<<1, 32>>>(out, cyc, n, 1.0000001); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("DFMA latency %.2f cyc\n", double(h) / n);
  lat_lds<<<1, 32>>>(out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("LDS latency %.2f cyc\n", double(h) / n);
  for (int t : {64, 256, 1024}) { syncthreads_cost<<<1, t>>>(cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("__syncthreads %d thr: %.2f cyc\n", t, double(h) / n); }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {1, 2, 4, 8, 16, 32}) {
    const int iters = 2048;
    thr_dadd<<<sms, 32 * warps>>>(out, iters, 1e-12);
    cudaEventRecord(e0); thr_dadd<<<sms, 32 * warps>>>(out, iters, 1e-12); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = double(sms) * 32 * warps * iters * 8;
    printf("DADD thr %2d warps/SM: %.1f Gop/s (%.1f lanes/clk/SM @1.965GHz)\n", warps, ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); thr_dfma<<<sms, 32 * warps>>>(out, iters, 1.0000001); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA thr %2d warps/SM: %.1f Gop/s (%.1f lanes/clk/SM)\n", warps, ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
