// Staging cost of a scorer tile: NC column slices of B bytes each (scattered
// sources in a 16 MB L2-resident buffer) copied into shared memory, per round,
// by (0) one cp.async.bulk per column issued by the lanes of warp 0, with one
// mbarrier transaction count, or (1) 16-byte cp.async (LDGSTS) spread over all
// 128 threads. Prints SM cycles per round (CTA 0) and the chip-wide rate, at
// 1..4 CTAs per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_issue.cu -o tma_issue
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(unsigned(__cvta_generic_to_shared(bar))), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(unsigned(__cvta_generic_to_shared(bar))),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
          unsigned(__cvta_generic_to_shared(bar))),
      "r"(parity));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   unsigned(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(bytes), "r"(unsigned(__cvta_generic_to_shared(bar)))
               : "memory");
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(unsigned(__cvta_generic_to_shared(dst))), "l"(src));
}

template <int MODE>
__global__ void __launch_bounds__(128) stage(const char* src, size_t ncol, int nc, int B, int iters, long long* cyc,
                                             double* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ unsigned long long bar;
  const int tid = threadIdx.x;
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  long long t0 = clock64();
  unsigned par = 0;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
      if (tid == 0) mbar_expect_tx(&bar, unsigned(nc * B));
      __syncwarp();
      if (tid < nc) {
        const size_t col = (size_t(blockIdx.x) * 7919 + size_t(it) * 131 + size_t(tid) * 977) % ncol;
        bulk_g2s(sm + tid * B, src + col * 4096, unsigned(B), &bar);
      }
      mbar_wait(&bar, par);
      par ^= 1;
    } else {
      const int chunks = nc * B / 16;
      for (int i = tid; i < chunks; i += 128) {
        const int c = i / (B / 16), u = i % (B / 16);
        const size_t col = (size_t(blockIdx.x) * 7919 + size_t(it) * 131 + size_t(c) * 977) % ncol;
        cp16(sm + c * B + u * 16, src + col * 4096 + u * 16);
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    acc += reinterpret_cast<const double*>(sm)[tid];
    __syncthreads();
  }
  if (tid == 0 && blockIdx.x == 0) *cyc = (clock64() - t0) / iters;
  if (acc == 1234.5) *sink = acc;
}

int main() {
  const size_t bytes = size_t(16) << 20;
  char* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 0, bytes);
  long long* cyc;
  double* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(stage<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  cudaFuncSetAttribute(stage<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int mode = 0; mode < 2; ++mode)
    for (int per_sm : {1, 3})
      for (int nc : {8, 16, 32})
        for (int B : {256, 512, 1024}) {
          if (nc * B > (48 << 10)) continue;
          const int grid = 148 * per_sm;
          auto k = mode == 0 ? stage<0> : stage<1>;
          k<<<grid, 128, nc * B>>>(src, bytes / 4096, nc, B, 10, cyc, sink);
          cudaEventRecord(e0);
          k<<<grid, 128, nc * B>>>(src, bytes / 4096, nc, B, iters, cyc, sink);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          long long c = 0;
          cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
          const double gbs = double(grid) * iters * nc * B / (ms * 1e-3) / 1e9;
          std::printf("%s ctas/sm %d cols %2d bytes %4d: %6lld cycles/round (CTA0), chip %7.0f GB/s %s\n",
                      mode == 0 ? "bulk  " : "ldgsts", per_sm, nc, B, c, gbs, cudaGetErrorString(cudaGetLastError()));
        }
  return 0;
}
