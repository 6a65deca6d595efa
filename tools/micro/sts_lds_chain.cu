// Single-warp round trip of the backward sweep's dependency: a lane stores a
// value to shared memory, the warp syncs, another lane loads it and runs the
// two complex products. Cycles per round for: the full chain, the chain
// without the shared round trip (register-carried), and the bare
// STS -> syncwarp -> LDS trip.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false sts_lds_chain.cu -o sts_lds_chain
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ double2 lds2(unsigned a) {
  double x, y;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
  return make_double2(x, y);
}
__device__ __forceinline__ void sts2(unsigned a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

template <int MODE>
__global__ void chain(int rounds, double2* out, long long* cyc) {
  __shared__ double2 x[64];
  const int lane = threadIdx.x;
  x[lane] = make_double2(1.0 + lane, 0.5);
  x[lane + 32] = make_double2(0.0, 0.0);
  __syncwarp();
  const unsigned xs = unsigned(__cvta_generic_to_shared(x));
  const double2 aa = make_double2(0.9, 0.01), pv = make_double2(1.01, -0.02), t = make_double2(0.3, 0.1);
  double2 reg = x[lane];
  const long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    // round r: lane reads the value lane-1 wrote in round r-1 (a chain across lanes)
    const int src = (lane + 31) & 31;
    double2 xj;
    if (MODE == 1)
      xj = reg;  // register-carried
    else
      xj = lds2(xs + 16u * unsigned(src));
    const double2 acc = make_double2(__dadd_rn(0.0, cmul(aa, xj).x), __dadd_rn(0.0, cmul(aa, xj).y));
    const double2 c = cmul(pv, acc);
    double2 res = make_double2(__dsub_rn(t.x, __dadd_rn(0.0, c.x)), __dsub_rn(t.y, __dadd_rn(0.0, c.y)));
    if (MODE == 2) res = xj;  // bare trip: no arithmetic
    if (MODE == 1)
      reg = res;
    else
      sts2(xs + 16u * unsigned(lane), res);
    if (MODE != 3) __syncwarp();
  }
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
  out[lane] = MODE == 1 ? reg : x[lane];
}

int main() {
  double2* out;
  long long* cyc;
  cudaMalloc(&out, 64 * sizeof(double2));
  cudaMalloc(&cyc, sizeof(long long));
  const char* names[] = {"STS->syncwarp->LDS + 2 cmul chain", "register-carried 2 cmul chain",
                         "bare STS->syncwarp->LDS", "STS->LDS chain without syncwarp"};
  const int rounds = 2000;
  for (int m = 0; m < 4; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) chain<0><<<1, 32>>>(rounds, out, cyc);
      if (m == 1) chain<1><<<1, 32>>>(rounds, out, cyc);
      if (m == 2) chain<2><<<1, 32>>>(rounds, out, cyc);
      if (m == 3) chain<3><<<1, 32>>>(rounds, out, cyc);
    }
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    std::printf("%-38s %6.1f cycles/round\n", names[m], double(c) / rounds);
  }
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
