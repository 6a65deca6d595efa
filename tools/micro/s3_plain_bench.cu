// Single-warp and per-SM cycle cost of the scorer's plain-row pass
// (s3_plain<1, 8>, kernels_score3.cuh) with its operands already in shared
// memory: no staging, no barriers. Separates the row arithmetic's own
// latency/throughput from the tile pipeline around it.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++20 \
//   -I../../include -I../../paper_2510_19608_b200/csrc s3_plain_bench.cu -o s3_plain_bench
#include <cuda_runtime.h>

#include <cstdio>

#include "kr_device.cuh"
#include "kr_internal.hpp"
namespace kronred::b200 {
using dev::C2;
}
#include "kernels_elim.cuh"
#include "kernels_csolve.cuh"
#include "kernels_score.cuh"
#include "kernels_score3.cuh"

using namespace kronred::b200;

template <int NRT>
__global__ void bench(int tiles, double* sink, long long* cyc) {
  constexpr int Ls = 8, RS = 2 * Ls;
  __shared__ double2 bv[K3 * RS];
  __shared__ double2 z[4 * (2 * K3 + 1)];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < K3 * RS; i += blockDim.x)
    bv[i] = make_double2(0.9 + 1e-3 * (i % 7), (i & 1) ? 0.95 : 0.91);
  for (int i = tid; i < 4 * (2 * K3 + 1); i += blockDim.x) z[i] = make_double2(1e-3 * (i % 5), -2e-3 * (i % 3));
  __syncthreads();
  const int gl = (lane / Ls) & 3, ll = lane % Ls;
  const double2* bvp = bv + ll;
  const double2* zp = z + gl * (2 * K3 + 1);
  C2 cv[1] = {{1e-2 + 1e-5 * tid, -3e-3}};
  double smice = 0, cm = 0, mx = 0;
  const long long t0 = clock64();
  for (int j = 0; j < tiles; ++j) {
#pragma unroll 1
    for (int hh = 0; hh < K3 / NRT; ++hh) s3_plain<1, NRT>(bvp, zp, RS, NRT * hh, cv, smice, cm, mx);
  }
  const long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + tid] = smice + mx;
}

int main() {
  double* sink;
  long long* cyc;
  cudaMalloc(&sink, 148 * 1024 * sizeof(double));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int tiles = 256;
  for (int warps : {1, 2, 3, 4, 8, 12, 16}) {
    for (int rep = 0; rep < 2; ++rep) bench<8><<<148, 32 * warps>>>(tiles, sink, cyc);
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    std::printf("NRT=8 warps/SM %2d: %6.1f cycles per row per warp, %6.1f SM-cycles per warp-row\n", warps,
                double(c) / (tiles * K3), double(c) / (tiles * K3) / warps);
  }
  for (int warps : {1, 4, 12}) {
    for (int rep = 0; rep < 2; ++rep) bench<4><<<148, 32 * warps>>>(tiles, sink, cyc);
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    std::printf("NRT=4 warps/SM %2d: %6.1f cycles per row per warp, %6.1f SM-cycles per warp-row\n", warps,
                double(c) / (tiles * K3), double(c) / (tiles * K3) / warps);
  }
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
