// Per-level cost of a warp-synchronous pull step: LDS -> complex chain -> STS -> __syncwarp.
#include <cstdio>
#include <cuda_runtime.h>
struct C2 { double x, y; };
__device__ __forceinline__ C2 cmul(C2 a, C2 b) { return {__dsub_rn(__dmul_rn(a.x,b.x), __dmul_rn(a.y,b.y)), __dadd_rn(__dmul_rn(a.x,b.y), __dmul_rn(a.y,b.x))}; }
__device__ __forceinline__ C2 cadd(C2 a, C2 b) { return {__dadd_rn(a.x,b.x), __dadd_rn(a.y,b.y)}; }
__device__ __forceinline__ C2 csub(C2 a, C2 b) { return {__dsub_rn(a.x,b.x), __dsub_rn(a.y,b.y)}; }
__global__ void k(long long* out, int levels, int variant) {
  extern __shared__ double2 dyn[];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* x = dyn + warp * 1024;
  double2* cf = dyn + 8 * 1024;
  int4* rec = reinterpret_cast<int4*>(cf + 1024);
  for (int i = lane; i < 1024; i += 32) { x[i] = make_double2(1.0 + i, 0.5); cf[i] = make_double2(0.999, 0.001); }
  for (int i = lane; i < 32 * 32; i += 32) rec[i] = make_int4((i * 37) & 1023, (i * 11) & 1023, (i * 29) & 1023, (i * 13) & 1023);
  __syncwarp();
  long long t0 = clock64();
  int4 rc = rec[lane];
  for (int lev = 0; lev < levels; ++lev) {
    int4 nx = rec[((lev + 1) & 31) * 32 + lane];
    if (variant == 0 || lane < 8) {
      double2 a0 = cf[rc.w], a1 = x[rc.z], xb = x[rc.x], p = cf[rc.y];
      C2 acc = cadd(C2{0,0}, cmul(C2{a0.x,a0.y}, C2{a1.x,a1.y}));
      C2 b = csub(C2{xb.x,xb.y}, acc);
      C2 t = cadd(C2{0,0}, cmul(C2{p.x,p.y}, b));
      x[rc.x] = make_double2(t.x, t.y);
    }
    rc = nx;
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
  long long* d; cudaMalloc(&d, 8); long long h;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int w : {1, 2, 4, 8})
  for (int v = 0; v < 2; ++v) {
    k<<<1, 32 * w, 9 * 1024 * 16 + 1024 * 16>>>(d, 1000, v); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("warps %d variant %d: %.1f cycles per level (%s)\n", w, v, h / 1000.0, cudaGetErrorString(cudaGetLastError()));
  }
}
