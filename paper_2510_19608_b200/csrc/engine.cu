// engine.cu — sm_100a kernels and the device side of run_reduction.
//
// Kernels (SURVEY §2 "native components"):
//   K1f  elim_factor_kernel   level-scheduled block elimination: structural
//                             pseudo-inverse pivots, Schur contributions
//                             (A_ik pinv_k) A_kj into slots, ordered apply.
//                             Serves the anchored factorization
//                             (solver.cpp:20-117, 168-179) and kron_reduce
//                             (kron.cpp:34-46, Y_kk - Y_kr Y_rr^-1 Y_rk).
//   K1s  csolve_kernel<MODE>  pull-form forward/backward sweeps on the
//                             present-phase compacted factor staged in shared
//                             memory (solver.cpp:119-148): scenario voltages,
//                             v0, the per-iteration base refresh
//                             (reduce.cpp:265) and the unit-injection Z
//                             columns (reduce.cpp:272).
//   K2/3 score_kernel         delta voltage Vc = base + sum_p c_p (Zs_p - Zr_p),
//                             |Vc|, voltage-margin feasibility and the ordered
//                             SMICE scan (reduce.cpp:80-123, 194-244).
//   K4   argmin_kernel        feasibility-masked lexicographic (smice, idx)
//                             argmin, warp shuffle then block (reduce.cpp:397-404).
//        commit_kernel        i_agg move + cluster bound merge (reduce.cpp:336-343).
//
// Exactness: see kr_device.cuh. Every decision is bit-identical to the
// reference CPU program (tests/test_gpu_parity.py).
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <set>
#include <stdexcept>
#include <atomic>
#include <functional>
#include <thread>

#include "kr_device.cuh"
#include "kr_internal.hpp"

namespace kronred::b200 {

using dev::C2;

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) ck((x), #x)

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) count = 1;
    CK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
};

}  // namespace
}  // namespace kronred::b200

#include "kernels_elim.cuh"
#include "kernels_csolve.cuh"
#include "kernels_score.cuh"
#include "kernels_score3.cuh"
#include "kernels_score1.cuh"
#include "kernels_loop.cuh"
#include "kernels_naive.cuh"

namespace kronred::b200 {
namespace {

// Unfused FP64 op-rate probe: 8 independent DMUL->DADD chains per thread.
__global__ void __launch_bounds__(256) fp64_probe_kernel(int iters, double a, double b, double* sink) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), b);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) sink[0] = s;
}

__global__ void selftest_cdiv_kernel(int N, const double* in, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const C2 r = dev::cdiv({in[4 * i], in[4 * i + 1]}, {in[4 * i + 2], in[4 * i + 3]});
  out[2 * i] = r.x;
  out[2 * i + 1] = r.y;
}

int gcd_int(int a, int b) { return b == 0 ? a : gcd_int(b, a % b); }

}  // namespace

// ---------------------------------------------------------------------------
// one elimination: schedule, device work lists, factor, compacted solve program

struct DevElim {
  ElimSchedule h;
  DBuf<int> ints;
  std::vector<size_t> off;  // offsets of each int array in `ints`
  DBuf<double2> blocks, pinv, contrib;
  DBuf<std::uint8_t> mask;
  DBuf<unsigned long long> fail;
  DBuf<double> fail_pivot;
  // present-phase compacted factor + level program for csolve_kernel
  CProg prog{};
  DBuf<int> meta;
  DBuf<long long> gsrc;
  DBuf<double2> cfac;
  DBuf<int> prow_off, prow_node;
  DBuf<std::uint8_t> prow_phase;
  std::vector<int> xoff;
  int smem_bytes = 0, smem_factor = 0;
  int wwarps = 0, wsm_factor = 0, wsmem_bytes = 0;
  int ncf_all = 0;  // gathered coefficients (program + padding entries)
  // lane-slot base-refresh program (base_refresh_kernel)
  BaseArgs bprog{};
  DBuf<int> bmeta;
  int bW = 0, bsmem = 0;
  bool bsm = true;  // factor + program staged in shared memory (else read from global)
  const int* P(int which) const { return ints.p + off[size_t(which)]; }
};

enum IntArr {
  A_STEP_NODE, A_STEP_DIAG, A_LVL_STEP_OFF, A_LVL_STEPS, A_LVL_SLOT_OFF, A_LVL_SLOTS,
  A_LVL_SLOT_STEP, A_SLOT_FROM, A_SLOT_TO, A_LVL_APPLY_OFF, A_APPLY_BLK, A_APPLY_OFF,
  A_APPLY_SLOTS, A_COUNT
};

constexpr int kTabPad = kTabPadRows;
#ifndef KRONRED_LOOP_UNROLL
#define KRONRED_LOOP_UNROLL 8
#endif
constexpr int kLoopUnroll = KRONRED_LOOP_UNROLL;  // loop iterations per conditional-graph body

struct Engine::Impl {
  Problem prob;
  int device = 0;
  cudaStream_t stream = nullptr;
  long long launches = 0;
  int n = 0, L = 0, nphi = 0;
  int optin_smem = 0;
  std::vector<int> prow_off, prow_node;
  std::vector<std::uint8_t> prow_phase;
  DBuf<int> d_prow_off, d_prow_node;
  DBuf<std::uint8_t> d_prow_phase, d_mask;
  DBuf<double2> d_yin;        // assembled Y blocks (input, resident)
  double pivot_floor = 0;
  DevElim full;               // anchored factorization of Y
  DBuf<double2> d_inj, d_vhat, d_v0, d_v0p, d_vhatp, d_iagg, d_iaggp, d_bv, d_Z, d_slackv;
  DBuf<double2> d_tfwd;  // [L][nphi] forward values of the last base refresh
  bool force_full_refresh = std::getenv("KRONRED_FULL_REFRESH") != nullptr;
  std::vector<double> h_vhat;  // [L][3n][2]
  // per-iteration inputs (pinned staging)
  DBuf<int4> d_cand;
  DBuf<unsigned> d_snt;
  DBuf<int> d_snid, d_memoff, d_memlist, d_snpos, d_memtmp;
  int4* h_cand = nullptr;
  unsigned* h_snt = nullptr;
  // magnitude path: active-row table + candidates grouped by |phi(r)|
  DBuf<unsigned> d_tab;
  DBuf<std::uint8_t> d_tplain;  // per 16-row tile: plain flag (score3)
  std::vector<std::uint8_t> h_tplain;
  DBuf<int> d_cidx;
  unsigned* h_tab = nullptr;
  int* h_cidx = nullptr;
  std::vector<int> tab_of_node;
  int R = 0;
  int grp_off[4] = {0, 0, 0, 0};
  std::vector<int> sn_pos;     // compact index of each active super-node
  DBuf<double> d_psmice, d_pmaxerr, d_pcand, d_best;
  // final Kron / model-error solves reuse these (no cudaMalloc/cudaFree inside a run)
  DevElim kron_e, merr_e;
  DBuf<double2> merr_yin, merr_rhs, merr_out, merr_kv;
  DBuf<int> d_grpdone;  // score3 slice-completion counters
  // score3 geometry: 16 Z-column slots per CTA, scenario slices of up to 8
  // scorer geometry: Z-column slots per CTA and scenario-slice width
  // (KRONRED_S3_G / KRONRED_S3_LS: tuning overrides, slots x width <= 128)
  // (with one or two scenarios a CTA is a single warp: twice the slots keep
  // two warps per CTA; 8,381 nodes x 2 scenarios 10.0 -> 9.0 s)
  int s3_slots() const {
    if (const char* e = std::getenv("KRONRED_S3_G")) {
      const int g = std::atoi(e);
      if (g < 3 || g > 128) throw ConfigError("KRONRED_S3_G must lie in [3, 128]");
      return g;
    }
    return L <= 2 ? 32 : 16;
  }
  // row split (lanes per pair): KRONRED_S3_S forces 1/2/4; otherwise the widest
  // split that keeps pairs x lanes within KRONRED_S3_FILL threads (default one
  // wave of 3 resident 128-thread CTAs on every SM)
  const int s3_force = std::getenv("KRONRED_S3_S") ? std::atoi(std::getenv("KRONRED_S3_S")) : 0;
  long long s3_fill() const {
    if (const char* e = std::getenv("KRONRED_S3_FILL")) return std::atoll(e);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    // score1 (small networks): split once pairs x lanes fit one wave of 3
    // resident CTAs per SM; score3 on large networks: about one CTA per SM,
    // with one or two scenarios 7/8 of one wave of the S = 2 launch (its CTAs
    // stage half the Z slots, so more fit per SM; 8,381 / 5,991 nodes x 2
    // scenarios: 8.9 -> 8.2 s / 4.5 -> 3.8 s, tools/s3fill_ab.sh)
    if (s1_ok()) return (long long)sms * 3 * 128;
    if (L <= 2) {
      int oc = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, score3_kernel<0>, s3_threads(),
                                                       S3Layout{s3_ls(), s3_slots(), 2, S3_NS_SPLIT}.smem_bytes()));
      return std::max(1LL, (long long)sms * oc * s3_threads() * 7 / 8);
    }
    return (long long)sms * 128;
  }
  // S = 4 starts at this many sixteenths of the fill: with one or two scenarios
  // on a large network at 14 (S = 4 wins below ~3/4 of its own wave: C4 / C3
  // L = 2 per-bucket sweep, tools/s3fill4_ab.sh), otherwise S3_FILL4_16
  int s3_fill4_16() const {
    if (const char* e = std::getenv("KRONRED_S3_FILL4")) return std::atoi(e);
    return !s1_ok() && L <= 2 ? 14 : S3_FILL4_16;
  }
  // slice-completion counters: one per candidate group at the widest split
  size_t s3_groups_max() const {
    size_t g = 8;
    for (int k = 1; k <= 3; ++k) g += size_t(s3_ldc() + s3_cpc(s3_slots(), k, 4) - 1) / size_t(s3_cpc(s3_slots(), k, 4));
    return g;
  }
  const int kS3Ls = std::getenv("KRONRED_S3_LS") ? std::atoi(std::getenv("KRONRED_S3_LS")) : 8;
  int s3_ls() const { return std::min(L, kS3Ls); }
  int s3_ldc() const { return std::max(2 * n, 2 * int(prob.net.branches.size()) + 1); }
  int s3_nsl() const { return (L + s3_ls() - 1) / s3_ls(); }
  int s3_threads() const {
    const int t = (s3_slots() * s3_ls() + 31) / 32 * 32;
    if (t > 128) throw ConfigError("scorer geometry: slots x slice width must not exceed 128 threads");
    return t;
  }
  S3Args s3_args() const {
    S3Args q{};
    q.L = L;
    q.nphi = nphi;
    q.G = s3_slots();
    q.S = 1;
    q.s_multi = s3_multi_lanes();
    q.Ls = s3_ls();
    q.nsl = s3_nsl();
    q.cand = d_cand.p;
    q.cand_idx = d_cidx.p;
    q.tab = d_tab.p;
    q.mask = d_mask.p;
    q.prow_off = d_prow_off.p;
    q.Z = d_Z.p;
    q.bv = d_bv.p;
    q.iagg = d_iagg.p;
    q.out_sm = d_psmice.p;
    q.out_mx = d_pmaxerr.p;
    q.ldc = s3_ldc();
    q.e_bar = cfg.e_bar;
    q.out_cand = d_pcand.p;
    q.grp_done = d_grpdone.p;
    q.tplain = d_tplain.p;
    return q;
  }

  // score1 (kernels_score1.cuh) takes the |phi(r)| = 1 candidates when the
  // scorer runs its default geometry (16 slots, slices of 8 scenarios)
  // (small networks: Z L2-resident; on large ones the wider score3 items
  // share more staging and measure faster: tools/large_ab.py)
  bool s1_ok() const {
    if (std::getenv("KRONRED_NO_S1")) return false;
    const bool fits = size_t(nphi) * size_t(nphi) * 16 <= (size_t(64) << 20) || std::getenv("KRONRED_FORCE_S1");
    return s3_ls() == kS1Ls && s3_slots() == kS1G && L <= 128 && fits;
  }
  // candidates per score1 item at S = 1, 2, 4 (KRONRED_S1_GK="8,8,4" tuning;
  // supported: 16/8 at S = 1 and 2, 8/4 at S = 4)
  int s1_gk[3] = {8, 8, 4};
  void parse_s1_gk() {
    if (const char* e = std::getenv("KRONRED_S1_GK")) {
      int a = 16, b = 8, c = 4;
      if (std::sscanf(e, "%d,%d,%d", &a, &b, &c) == 3 && (a == 16 || a == 8) && (b == 16 || b == 8) && (c == 8 || c == 4)) {
        s1_gk[0] = a;
        s1_gk[1] = b;
        s1_gk[2] = c;
      } else {
        throw ConfigError("KRONRED_S1_GK: three of 16|8, 16|8, 8|4");
      }
    }
  }
  template <int S, int GK>
  void launch_s1_k(const S3Args& q, int grid, cudaStream_t st) {
    constexpr size_t sm = s1_smem_bytes<S, GK>();
    if (sm > 48 * 1024)  // (tuning geometries with a deep ring)
      CK(cudaFuncSetAttribute(score1_kernel<S, GK>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    score1_kernel<S, GK><<<grid, S1Geom<S, GK>::P, sm, st>>>(q);
  }
  void launch_s1(int S, const S3Args& q, int grid, cudaStream_t st) {
    if (grid <= 0) return;
    const int gk = s1_gk[s1_switch_index(S)];
    if (S == 1)
      gk == 16 ? launch_s1_k<1, 16>(q, grid, st) : launch_s1_k<1, 8>(q, grid, st);
    else if (S == 2)
      gk == 16 ? launch_s1_k<2, 16>(q, grid, st) : launch_s1_k<2, 8>(q, grid, st);
    else
      gk == 8 ? launch_s1_k<4, 8>(q, grid, st) : launch_s1_k<4, 4>(q, grid, st);
    launched();
    CK(cudaGetLastError());
  }
  // occupancy-sized persistent grid of the score1 variant for split S
  int s1_grid(int S, int items_max) {
    const int gk = s1_gk[s1_switch_index(S)];
    int occ = 0;
    auto occ_of = [&](auto kern, int P, size_t sm) {
      if (sm > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, P, sm));
    };
    if (S == 1)
      gk == 16 ? occ_of(score1_kernel<1, 16>, 128, s1_smem_bytes<1, 16>()) : occ_of(score1_kernel<1, 8>, 64, s1_smem_bytes<1, 8>());
    else if (S == 2)
      gk == 16 ? occ_of(score1_kernel<2, 16>, 256, s1_smem_bytes<2, 16>()) : occ_of(score1_kernel<2, 8>, 128, s1_smem_bytes<2, 8>());
    else
      gk == 8 ? occ_of(score1_kernel<4, 8>, 256, s1_smem_bytes<4, 8>()) : occ_of(score1_kernel<4, 4>, 128, s1_smem_bytes<4, 4>());
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    return std::max(1, std::min(items_max * 2, std::max(1, occ) * sms));
  }
  static int s1_switch_index(int S) { return S == 1 ? 0 : (S == 2 ? 1 : 2); }
  // split of the |phi(r)| >= 2 candidates next to score1 (KRONRED_S3_MULTI)
  int s3_multi_lanes() const {
    const int v = std::getenv("KRONRED_S3_MULTI") ? std::atoi(std::getenv("KRONRED_S3_MULTI")) : 4;
    return (v == 1 || v == 2 || v == 4) ? v : 4;
  }

  // threads per scorer CTA: a multiple of L (whole candidates) and of 32
  int score_cta_threads() const {
    int P = L * (32 / gcd_int(L, 32));
    if (P > 256) P = (L + 31) / 32 * 32;  // one candidate per CTA, idle tail lanes
    if (P > 512) throw ConfigError("more than 512 scenarios are not supported by the scorer CTA layout");
    return P;
  }
  double* h_best = nullptr;    // pinned [2 + L]
  size_t h_best_n = 0;
  // multi-GPU
  int rank = 0, world = 1;
  krg_exchange_fn xfn = nullptr;
  void* xuser = nullptr;
  // in-graph exchange: NCCL communicator, symmetric window of per-rank records
  // (2 parities x world x rec_bytes), device communicator with one LSA barrier
  ncclComm_t comm = nullptr;
  ncclWindow_t win = nullptr;
  void* winbuf = nullptr;
  ncclDevComm dcomm{};
  int rec_bytes = 0, xemul = 1;
  static void nk(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(std::string("NCCL error in ") + what + ": " + ncclGetErrorString(r));
  }
  void set_comm(int rk, int ws, const ncclUniqueId& id) {
    if (ws < 1 || rk < 0 || rk >= ws) throw ConfigError("bad rank/world");
    free_comm();
    CK(cudaSetDevice(device));
    nk(ncclCommInitRank(&comm, ws, id, rk), "ncclCommInitRank");
    rec_bytes = (24 + 8 * std::max(L, 1) + 15) & ~15;
    // test aid: a one-rank communicator playing KRONRED_XCH_EMULATE ranks
    xemul = ws == 1 && std::getenv("KRONRED_XCH_EMULATE") ? std::max(1, std::atoi(std::getenv("KRONRED_XCH_EMULATE"))) : 1;
    const size_t bytes = (size_t(2) * std::max(ws, xemul) * rec_bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) /
                         NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    nk(ncclMemAlloc(&winbuf, bytes), "ncclMemAlloc");
    nk(ncclCommWindowRegister(comm, winbuf, bytes, &win, NCCL_WIN_COLL_SYMMETRIC), "ncclCommWindowRegister");
    ncclDevCommRequirements req{};
    req.lsaBarrierCount = 1;
    nk(ncclDevCommCreate(comm, &req, &dcomm), "ncclDevCommCreate");
    rank = rk;
    world = ws;
  }
  void free_comm() {
    if (!comm) return;
    ncclDevCommDestroy(comm, &dcomm);
    ncclCommWindowDeregister(comm, win);
    ncclMemFree(winbuf);
    ncclCommDestroy(comm);
    comm = nullptr;
    win = nullptr;
    winbuf = nullptr;
  }
  // loop state
  ReductionConfig cfg;
  HostState hs;
  std::vector<int> cs, cr;
  bool loop_active = false;
  // kernel statistics (enabled on demand; CUDA events on the launching stream)
  bool profile = false;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_run0 = nullptr, ev_run1 = nullptr;
  KernelStats score_stats{}, solve_stats{}, multi_stats{};
  long long score_c0 = 0;
  // device-resident loop (kernels_loop.cuh)
  DBuf<LoopState> d_loopst;
  DBuf<int> d_sup, d_sn, d_tabnode, d_cs, d_cr, d_brf, d_brt, d_trsr, d_trc;
  DBuf<double> d_trsmice, d_trme;
  DBuf<unsigned long long> d_trt;
  cudaStream_t stream2 = nullptr, stream3 = nullptr, stream_cap = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_fork3 = nullptr, ev_join3 = nullptr;
  // Inside a stream capture: a switch conditional node on `h` with three
  // bodies; body i is captured by launch(i, capture stream).
  template <class F>
  void add_switch(cudaStream_t st, cudaGraphConditionalHandle h, F&& launch) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    const cudaGraphEdgeData* ed = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo_v3(st, &cs, nullptr, &g, &deps, &ed, &nd));
    if (cs != cudaStreamCaptureStatusActive) throw Error("add_switch outside a capture");
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeSwitch;
    cp.conditional.size = 3;
    cudaGraphNode_t node;
    {
      const cudaError_t e = cudaGraphAddNode_v2(&node, g, deps, ed, nd, &cp);
      if (e != cudaSuccess) {
        std::string why = "add_switch: cudaGraphAddNode (" + std::to_string(nd) + " deps";
        for (size_t i = 0; ed && i < nd; ++i) why += ", edge type " + std::to_string(int(ed[i].type)) + " port " + std::to_string(int(ed[i].from_port));
        throw CudaError(why + "): " + cudaGetErrorString(e));
      }
    }
    if (!stream_cap) CK(cudaStreamCreateWithFlags(&stream_cap, cudaStreamNonBlocking));
    for (int i = 0; i < 3; ++i) {
      cudaGraph_t bg = cp.conditional.phGraph_out[i];
      CK(cudaStreamBeginCaptureToGraph(stream_cap, bg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      launch(i, stream_cap);
      CK(cudaStreamEndCapture(stream_cap, &bg));
    }
    CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  }
  // the loop graph is instantiated once per engine and configuration
  cudaGraph_t loop_graph = nullptr;
  cudaGraphExec_t loop_exec = nullptr;
  double loop_key_ebar = -1.0, loop_key_target = -1.0;
  int loop_key_has = -1;
  bool loop_key_trace = false;
  // buffers the captured graph refers to (a reload may reallocate them)
  static constexpr int kLoopKeyBufs = 18;
  const void* loop_key_bufs[kLoopKeyBufs] = {};
  int loop_key_L = -1;
  bool loop_key_live = false;
  bool last_device_loop = false;  // the last run() took the device-resident loop graph
  ncclComm_t loop_key_comm = nullptr;
  int loop_key_cplx = -1;
  DBuf<unsigned long long> d_tdbg;
  bool loop_trace = std::getenv("KRONRED_LOOP_TRACE") != nullptr;
  bool force_host_loop = std::getenv("KRONRED_LOOP") != nullptr && std::string(std::getenv("KRONRED_LOOP")) == "host";

  void launched() { ++launches; }

  void ensure_events() {
    if (!ev_a) {
      CK(cudaEventCreate(&ev_a));
      CK(cudaEventCreate(&ev_b));
      CK(cudaEventCreate(&ev_run0));
      CK(cudaEventCreate(&ev_run1));
    }
  }

  float event_ms() {
    CK(cudaEventRecord(ev_b, stream));
    CK(cudaEventSynchronize(ev_b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev_a, ev_b));
    return ms;
  }

  // algorithmic work of one score launch: flops and bytes
  // only: 0 every candidate, 1 those with |phi(r)| = 1, 2 those with |phi(r)| >= 2
  void score_work(long long c0, long long c1, double& flops, double& bytes, int only = 0) const {
    long long R = 0;
    for (int i : hs.supernodes) R += PhaseMask{prob.mask[size_t(i)]}.count();
    const long long ns = (long long)hs.supernodes.size();
    std::set<int> cols;
    flops = 0;
    long long nc = 0;
    for (long long c = c0; c < c1; ++c) {
      const int q = PhaseMask{prob.mask[size_t(cr[size_t(c)])]}.count();
      if ((only == 1 && q != 1) || (only == 2 && q == 1)) continue;
      ++nc;
      const double Rp = double(R - q);
      flops += 2.0 * q * Rp + double(L) * ((8.0 * q + 4.0) * Rp + 2.0 * nphi + double(ns - 1));
      cols.insert(cs[size_t(c)]);
      cols.insert(cr[size_t(c)]);
    }
    long long zc = 0;
    for (int node : cols) zc += PhaseMask{prob.mask[size_t(node)]}.count();
    bytes = 16.0 * double(zc) * double(R)               // Z columns of every endpoint over active rows
            + double(L) * double(R) * 32.0              // base + cluster min/max
            + double(nc) * (16.0 + 48.0 * L)            // candidates + i_agg of r
            + 4.0 * double(ns) + 16.0 * double(nc) * L;  // super-node table + outputs
  }

  // ---- elimination schedules -----------------------------------------------

  void upload_elim(DevElim& d, const FlatBlocks& y, const std::vector<std::uint8_t>& mask,
                   const std::vector<int>& elim, bool with_solve = true) {
    d.h = build_schedule(y, mask, elim);
    const ElimSchedule& h = d.h;
    const std::vector<const std::vector<int>*> arrs = {
        &h.step_node, &h.step_diag, &h.lvl_step_off, &h.lvl_steps, &h.lvl_slot_off, &h.lvl_slots,
        &h.lvl_slot_step, &h.slot_from, &h.slot_to, &h.lvl_apply_off, &h.apply_blk, &h.apply_off,
        &h.apply_slots};
    d.off.assign(A_COUNT + 1, 0);
    for (int i = 0; i < A_COUNT; ++i) d.off[size_t(i) + 1] = d.off[size_t(i)] + arrs[size_t(i)]->size();
    std::vector<int> packed(d.off[A_COUNT]);
    for (int i = 0; i < A_COUNT; ++i)
      std::copy(arrs[size_t(i)]->begin(), arrs[size_t(i)]->end(), packed.begin() + long(d.off[size_t(i)]));
    d.ints.alloc(packed.size());
    if (!packed.empty())
      CK(cudaMemcpyAsync(d.ints.p, packed.data(), packed.size() * sizeof(int), cudaMemcpyHostToDevice, stream));
    d.blocks.alloc(size_t(std::max(h.nblocks, 1)) * 9);
    d.pinv.alloc(size_t(std::max(h.nsteps, 1)) * 9);
    d.contrib.alloc(size_t(std::max(h.nslots, 1)) * 9);
    d.mask.alloc(mask.size());
    CK(cudaMemcpyAsync(d.mask.p, mask.data(), mask.size(), cudaMemcpyHostToDevice, stream));
    d.fail.alloc(1);
    d.fail_pivot.alloc(size_t(std::max(h.nsteps, 1)));
    CK(cudaStreamSynchronize(stream));
    if (with_solve) build_compact(d);
  }

  // Host: present-phase layout of the factor and the packed level program
  // (records in level order, see kernels_csolve.cuh).
  void build_compact(DevElim& d) {
    const ElimSchedule& h = d.h;
    const int nn = h.n;
    d.xoff.assign(size_t(nn) + 1, 0);
    for (int i = 0; i < nn; ++i) d.xoff[size_t(i) + 1] = d.xoff[size_t(i)] + __builtin_popcount(h.mask[size_t(i)]);
    const int nph = d.xoff[size_t(nn)];
    std::vector<int> pnode(size_t(std::max(nph, 1)), 0);
    std::vector<std::uint8_t> pphase(size_t(std::max(nph, 1)), 0);
    for (int i = 0; i < nn; ++i) {
      int t = d.xoff[size_t(i)];
      for (int p = 0; p < 3; ++p)
        if ((h.mask[size_t(i)] >> p) & 1) {
          pnode[size_t(t)] = i;
          pphase[size_t(t)] = std::uint8_t(p);
          ++t;
        }
    }
    std::vector<long long> g;
    auto present = [&](int node, int* idx) {
      int k = 0;
      for (int p = 0; p < 3; ++p)
        if ((h.mask[size_t(node)] >> p) & 1) idx[k++] = p;
      return k;
    };
    auto gather_block = [&](long long base9, bool is_pinv, int rn, int cn) {
      int ri[3], ci[3];
      const int mr = present(rn, ri), mc = present(cn, ci);
      const int off = int(g.size());
      for (int i = 0; i < mr; ++i)
        for (int j = 0; j < mc; ++j)
          g.push_back(base9 < 0 ? -1 : (((base9 + ri[i] * 3 + ci[j]) << 1) | (is_pinv ? 1 : 0)));
      return off;
    };
    auto xm = [&](int node) {
      const int m = __builtin_popcount(h.mask[size_t(node)]);
      if (d.xoff[size_t(node)] >= (1 << 24)) throw Error("solution vector too large for the packed program");
      return d.xoff[size_t(node)] | (m << 24);
    };
    // per-step factor offsets
    std::vector<int> pinv_off(size_t(h.nsteps)), fin_first(size_t(h.nsteps)), bcp_first(size_t(h.nsteps));
    std::vector<int> fin_x, fin_b, bcp_x, bcp_b;
    for (int st = 0; st < h.nsteps; ++st) {
      const int k = h.step_node[size_t(st)];
      pinv_off[size_t(st)] = gather_block((long long)st * 9, true, k, k);
      fin_first[size_t(st)] = int(fin_x.size());
      for (int e = h.in_off[size_t(st)]; e < h.in_off[size_t(st) + 1]; ++e) {
        const int j = h.in_node[size_t(e)], b = h.in_blk[size_t(e)];
        fin_x.push_back(xm(j));
        fin_b.push_back(gather_block(b < 0 ? -1 : (long long)b * 9, false, k, j));
      }
      bcp_first[size_t(st)] = int(bcp_x.size());
      for (int e = h.cpl_off[size_t(st)]; e < h.cpl_off[size_t(st) + 1]; ++e) {
        const int j = h.cpl_node[size_t(e)], b = h.cpl_to[size_t(e)];
        bcp_x.push_back(xm(j));
        bcp_b.push_back(gather_block(b < 0 ? -1 : (long long)b * 9, false, k, j));
      }
    }
    std::vector<int> meta;
    auto align4 = [&]() {
      while (meta.size() % 4) meta.push_back(0);
    };
    CProg P{};
    // forward records (level order) + their pull entries (contiguous per record)
    align4();
    P.frec = int(meta.size());
    std::vector<int> fent;
    for (int i = 0; i < h.nsteps && h.nsteps > 0; ++i) {
      const int st = h.fw_steps[size_t(i)];
      const int k = h.step_node[size_t(st)];
      const int ne = h.in_off[size_t(st) + 1] - h.in_off[size_t(st)];
      if (ne > 255) throw Error("elimination step has more than 255 pulls");
      bool scalar = __builtin_popcount(h.mask[size_t(k)]) == 1;
      for (int e = 0; e < ne; ++e) scalar = scalar && (fin_x[size_t(fin_first[size_t(st)] + e)] >> 24) == 1;
      meta.push_back(xm(k) | (int(h.mask[size_t(k)]) << 26) | (scalar ? (1 << 29) : 0));
      meta.push_back(k);
      meta.push_back(pinv_off[size_t(st)]);
      meta.push_back(int(fent.size() / 2) | (ne << 24));
      for (int e = 0; e < ne; ++e) {
        fent.push_back(fin_x[size_t(fin_first[size_t(st)] + e)]);
        fent.push_back(fin_b[size_t(fin_first[size_t(st)] + e)]);
      }
    }
    align4();
    P.fent = int(meta.size());
    meta.insert(meta.end(), fent.begin(), fent.end());
    align4();
    P.brec = int(meta.size());
    std::vector<int> bent;
    for (int i = 0; i < h.nsteps && h.nsteps > 0; ++i) {
      const int st = h.bw_steps[size_t(i)];
      const int k = h.step_node[size_t(st)];
      const int ne = h.cpl_off[size_t(st) + 1] - h.cpl_off[size_t(st)];
      if (ne > 255) throw Error("elimination step has more than 255 couplings");
      bool scalar = __builtin_popcount(h.mask[size_t(k)]) == 1;
      for (int e = 0; e < ne; ++e) scalar = scalar && (bcp_x[size_t(bcp_first[size_t(st)] + e)] >> 24) == 1;
      meta.push_back(xm(k) | (scalar ? (1 << 29) : 0));
      meta.push_back(k);
      meta.push_back(pinv_off[size_t(st)]);
      meta.push_back(int(bent.size() / 2) | (ne << 24));
      for (int e = 0; e < ne; ++e) {
        bent.push_back(bcp_x[size_t(bcp_first[size_t(st)] + e)]);
        bent.push_back(bcp_b[size_t(bcp_first[size_t(st)] + e)]);
      }
    }
    align4();
    P.bent = int(meta.size());
    meta.insert(meta.end(), bent.begin(), bent.end());
    P.fw_off = int(meta.size());
    if (h.nsteps > 0) meta.insert(meta.end(), h.fw_off.begin(), h.fw_off.end());
    P.bw_off = int(meta.size());
    if (h.nsteps > 0) meta.insert(meta.end(), h.bw_off.begin(), h.bw_off.end());
    P.kept = int(meta.size());
    for (size_t kk = 0; kk < h.kept.size(); ++kk) {
      meta.push_back(xm(h.kept[kk]));
      meta.push_back(int(kk));
    }
    align4();
    P.nsteps = h.nsteps;
    P.nfw = h.nsteps ? h.nfw : 0;
    P.nbw = h.nsteps ? h.nbw : 0;
    P.nkept = int(h.kept.size());
    P.nmeta = int(meta.size());
    P.ncf = int(g.size());
    P.nphi = nph;
    d.prog = P;
    {
      // lane-slot program: per level round 32 records, scalar one-entry steps inline
      std::vector<int> bm, fe2, be2;
      const int zero_cf = int(g.size());
      g.push_back(-1);  // one exact-zero coefficient for pull-free steps
      std::vector<int> frec_of_step(size_t(std::max(h.nsteps, 1)), -1);
      auto slots = [&](const std::vector<int>& off, const std::vector<int>& steps, bool fwd, int& nrounds,
                       std::vector<int>& recs, std::vector<int>& ext, std::vector<int>& ents, int lanes) {
        nrounds = 0;
        const int nl = h.nsteps ? int(off.size()) - 1 : 0;
        auto empty = [&]() {
          recs.insert(recs.end(), {-1, 0, 0, 0});
          ext.insert(ext.end(), {0, 0, 0, 0});
        };
        // lanes a backward general step takes: one per present phase (its rows
        // are independent until the pivot product, a shuffle apart) when the
        // round is one warp and KRONRED_NO_GEN_SPLIT is unset
        const bool split = !fwd && lanes == 32 && std::getenv("KRONRED_NO_GEN_SPLIT") == nullptr;
        auto demand = [&](int st) {
          if (!split) return 1;
          const int k = h.step_node[size_t(st)];
          const int mk = __builtin_popcount(h.mask[size_t(k)]);
          const int first = bcp_first[size_t(st)];
          const int ne = h.cpl_off[size_t(st) + 1] - h.cpl_off[size_t(st)];
          bool scalar = mk == 1;
          for (int e = 0; e < ne; ++e) scalar = scalar && (bcp_x[size_t(first + e)] >> 24) == 1;
          return scalar ? 1 : mk;
        };
        int gen_first = 0;
        auto emit = [&](int st, int row) {
          const int k = h.step_node[size_t(st)];
          const int mk = __builtin_popcount(h.mask[size_t(k)]);
          if (fwd) frec_of_step[size_t(st)] = int(recs.size() / 4);
          const int first = fwd ? fin_first[size_t(st)] : bcp_first[size_t(st)];
          const int ne = fwd ? h.in_off[size_t(st) + 1] - h.in_off[size_t(st)]
                             : h.cpl_off[size_t(st) + 1] - h.cpl_off[size_t(st)];
          const std::vector<int>& ex = fwd ? fin_x : bcp_x;
          const std::vector<int>& eb = fwd ? fin_b : bcp_b;
          bool scalar = mk == 1;
          for (int e = 0; e < ne; ++e) scalar = scalar && (ex[size_t(first + e)] >> 24) == 1;
          if (size_t(d.xoff[size_t(nn)]) * 16 >= (1u << 31) || size_t(g.size()) * 16 >= (1u << 31))
            throw Error("base program offsets overflow");
          if (scalar && fwd) {
            // forward: the first two pulls inline; missing pulls are exact
            // zero pulls (b - (0 + 0*x) == b bit for bit), so every scalar
            // step runs the same instruction sequence with both products
            // in flight at once
            const int xj = ne == 0 ? d.xoff[size_t(k)] : (ex[size_t(first)] & 0xffffff);
            const int bo = ne == 0 ? zero_cf : eb[size_t(first)];
            const int xj1 = ne < 2 ? d.xoff[size_t(k)] : (ex[size_t(first + 1)] & 0xffffff);
            const int bo1 = ne < 2 ? zero_cf : eb[size_t(first + 1)];
            recs.insert(recs.end(), {d.xoff[size_t(k)] * 16, pinv_off[size_t(st)] * 16, xj * 16, bo * 16});
            ext.insert(ext.end(), {xj1 * 16, bo1 * 16, int(ents.size() / 2), std::max(ne - 2, 0)});
            for (int e = 2; e < ne; ++e) {
              ents.push_back(ex[size_t(first + e)]);
              ents.push_back(eb[size_t(first + e)]);
            }
          } else if (scalar) {
            // backward: first coupling inline (an exact-zero one when none)
            const int xj = ne == 0 ? d.xoff[size_t(k)] : (ex[size_t(first)] & 0xffffff);
            const int bo = ne == 0 ? zero_cf : eb[size_t(first)];
            recs.insert(recs.end(), {d.xoff[size_t(k)] * 16, pinv_off[size_t(st)] * 16, xj * 16, bo * 16});
            ext.insert(ext.end(), {0, mk, int(ents.size() / 2), std::max(ne - 1, 0)});
            for (int e = 1; e < ne; ++e) {
              ents.push_back(ex[size_t(first + e)]);
              ents.push_back(eb[size_t(first + e)]);
            }
          } else {
            // general step; split over mk lanes (backward, row r per lane:
            // ext.x = 1 | 2 | r << 8), the coupling entries shared
            recs.insert(recs.end(), {d.xoff[size_t(k)] * 16, pinv_off[size_t(st)] * 16, fwd ? -1 : 0, 0});
            if (row <= 0) {
              gen_first = int(ents.size() / 2);
              for (int e = 0; e < ne; ++e) {
                ents.push_back(ex[size_t(first + e)]);
                ents.push_back(eb[size_t(first + e)]);
              }
            }
            ext.insert(ext.end(), {row < 0 ? 1 : (3 | (row << 8)), mk, gen_first, ne});
          }
        };
        for (int lv = 0; lv < nl; ++lv) {
          const int c0 = off[size_t(lv)], cnt = off[size_t(lv) + 1] - c0;
          for (int i = 0; i < cnt; ++nrounds) {
            int used = 0;
            while (i < cnt) {
              const int st = steps[size_t(c0 + i)];
              const int dm = demand(st);
              if (used + dm > lanes) break;
              for (int r = 0; r < dm; ++r) emit(st, dm > 1 ? r : -1);
              used += dm;
              ++i;
            }
            for (; used < lanes; ++used) empty();
          }
        }
        for (int ln = 0; ln < lanes; ++ln) empty();  // padding round for the unconditional prefetch
      };
      std::vector<int> frecs, brecs, fext, bext;
      int nfr = 0, nbr = 0;
      slots(h.fw_off, h.fw_steps, true, nfr, frecs, fext, fe2, 32);
      slots(h.bw_off, h.bw_steps, false, nbr, brecs, bext, be2, 32);
      // A program too large for shared memory (large feeders) runs from
      // global memory with one scenario per CTA; its backward sweep then
      // spreads each level over kRefreshWB warps (rounds of 32 * kRefreshWB
      // slots, a CTA barrier per round): wide levels take ~1 round, not
      // width / 32.
      int wb = 1;
      {
        const size_t est = (g.size() + 1) * 16 +
                           (frecs.size() + fext.size() + brecs.size() + bext.size() + fe2.size() + be2.size() +
                            size_t(nn) * 4 + 2 * h.kept.size() + 64) * 4;
        if (est + size_t(nph) * 16 > size_t(optin_smem) - 64 && std::getenv("KRONRED_REFRESH_WB1") == nullptr) {
          wb = kRefreshWB;
          brecs.clear();
          bext.clear();
          be2.clear();
          slots(h.bw_off, h.bw_steps, false, nbr, brecs, bext, be2, 32 * wb);
        }
      }
      BaseArgs& B = d.bprog;
      {
        // first backward round of an all-scalar suffix (tree_backward's tight loop)
        const int lanes = int(brecs.size() / 4) / std::max(nbr + 1, 1);
        int bf = nbr;
        for (int r = nbr - 1; r >= 0; --r) {
          bool fast = true;
          for (int l = 0; l < lanes && fast; ++l) {
            const size_t q = size_t(r * lanes + l) * 4;
            fast = brecs[q] < 0 || (bext[q] == 0 && bext[q + 3] == 0);
          }
          if (!fast) break;
          bf = r;
        }
        B.bfast = std::getenv("KRONRED_NO_BFAST") ? nbr : bf;
      }
      auto put4 = [&](const std::vector<int>& v) {
        while (bm.size() % 4) bm.push_back(0);
        const int o = int(bm.size());
        bm.insert(bm.end(), v.begin(), v.end());
        return o;
      };
      B.fslot = put4(frecs);
      B.bslot = put4(brecs);
      B.fext = put4(fext);
      B.bext = put4(bext);
      B.fent = put4(fe2);
      B.bent = put4(be2);
      std::vector<int> kp;
      for (size_t kk = 0; kk < h.kept.size(); ++kk) {
        kp.push_back(xm(h.kept[kk]));
        kp.push_back(int(kk));
      }
      B.kept = put4(kp);
      // incremental forward walk: per node {forward record, elimination-tree
      // parent, step index}; only for trees (every node feeds one later node)
      {
        std::vector<int> wk(size_t(nn) * 4, -1);
        bool tree = h.nsteps > 0;
        for (int st = 0; st < h.nsteps; ++st) {
          const int k = h.step_node[size_t(st)];
          wk[size_t(k) * 4 + 0] = frec_of_step[size_t(st)];
          wk[size_t(k) * 4 + 2] = st;
          for (int e = h.in_off[size_t(st)]; e < h.in_off[size_t(st) + 1]; ++e) {
            const int j = h.in_node[size_t(e)];
            if (wk[size_t(j) * 4 + 1] >= 0) tree = false;
            wk[size_t(j) * 4 + 1] = k;
          }
        }
        B.walk = tree ? put4(wk) : -1;
        if (tree && std::getenv("KRONRED_WALK_STATS")) {  // debugging aid: elimination-tree depth
          std::vector<int> dep(size_t(nn), 0);
          long long sum = 0;
          int mx = 0, cnt = 0;
          for (int st = h.nsteps - 1; st >= 0; --st) {
            const int k = h.step_node[size_t(st)], par = wk[size_t(k) * 4 + 1];
            dep[size_t(k)] = par >= 0 && wk[size_t(par) * 4] >= 0 ? dep[size_t(par)] + 1 : 1;
            sum += dep[size_t(k)];
            mx = std::max(mx, dep[size_t(k)]);
            ++cnt;
          }
          std::fprintf(stderr, "walk: %d steps, depth mean %.1f max %d, levels %d\n", cnt, double(sum) / std::max(cnt, 1), mx, nbr);
          const int lanes = int(brecs.size() / 4) / std::max(nbr + 1, 1);
          for (int r = 0; r < nbr; ++r)
            for (int l = 0; l < lanes; ++l) {
              const size_t q = size_t(r * lanes + l) * 4;
              if (brecs[q] < 0 || bext[q] == 0) continue;
              std::fprintf(stderr, "  backward round %d lane %d: general mk %d couplings %d:", r, l, bext[q + 1], bext[q + 3]);
              for (int e = 0; e < bext[q + 3]; ++e) std::fprintf(stderr, " mj%d", be2[size_t(bext[q + 2] + e) * 2] >> 24);
              std::fprintf(stderr, "\n");
            }
          for (int st = 0; st < h.nsteps; ++st) {
            const int k = h.step_node[size_t(st)];
            const int q = frec_of_step[size_t(st)] * 4;
            if (frecs[size_t(q) + 2] >= 0) continue;
            std::fprintf(stderr, "  forward step %d node %d: general mk %d pulls %d depth %d\n", st, k, fext[size_t(q) + 1],
                         fext[size_t(q) + 3], dep[size_t(k)]);
          }
        }
      }
      while (bm.size() % 4) bm.push_back(0);
      B.nfr = nfr;
      B.nbr = nbr;
      B.nkept = int(h.kept.size());
      B.nmeta = int(bm.size());
      B.ncf = int(g.size());
      B.nphi = nph;
      d.bmeta.alloc(bm.size());
      CK(cudaMemcpyAsync(d.bmeta.p, bm.data(), bm.size() * sizeof(int), cudaMemcpyHostToDevice, stream));
      const size_t fixed = size_t(B.ncf) * 16 + size_t(B.nmeta) * 4;
      d.bW = 0;
      d.bsm = true;
      B.rhs_staged = B.walk >= 0 ? 1 : 0;
      // two nph-row buffers per warp when the incremental walk is available
      size_t per_warp = size_t(nph) * 16 * (B.walk >= 0 ? 2 : 1);
      for (int w = 8; w >= 1; --w)
        if (fixed + size_t(w) * per_warp <= size_t(optin_smem) - 64) {
          d.bW = w;
          break;
        }
      size_t fx = fixed;
      B.WB = 1;
      if (wb > 1) d.bW = 0;  // global program, one scenario per CTA
      if (d.bW == 0 && wb > 1) {
        d.bsm = false;
        fx = 0;
        B.WB = wb;
        per_warp = size_t(nph) * 16 * (B.walk >= 0 ? 2 : 1);
        B.rhs_staged = B.walk >= 0 ? 1 : 0;
        if (per_warp > size_t(optin_smem) - 64) {
          per_warp = size_t(nph) * 16;
          B.rhs_staged = 0;
        }
        d.bW = 1;
      }
      if (d.bW == 0) {
        // large network: factor and program stay in global memory (read
        // through L1/L2); only the solution (and, if they fit, the staged
        // right-hand sides) live in shared memory
        d.bsm = false;
        fx = 0;
        for (int stage = 1; stage >= 0 && d.bW == 0; --stage) {
          per_warp = size_t(nph) * 16 * (B.walk >= 0 && stage ? 2 : 1);
          for (int w = 8; w >= 1; --w)
            if (size_t(w) * per_warp <= size_t(optin_smem) - 64) {
              d.bW = w;
              B.rhs_staged = B.walk >= 0 && stage ? 1 : 0;
              break;
            }
        }
      }
      if (const char* e = std::getenv("KRONRED_REFRESH_W"))  // tuning aid: cap scenario warps per CTA
        d.bW = std::max(1, std::min(d.bW, std::atoi(e)));
      d.bsmem = int(fx + size_t(std::max(d.bW, 1)) * per_warp);
    }
    d.meta.alloc(meta.size());
    if (!meta.empty())
      CK(cudaMemcpyAsync(d.meta.p, meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice, stream));
    d.ncf_all = int(g.size());
    d.gsrc.alloc(g.size());
    if (!g.empty())
      CK(cudaMemcpyAsync(d.gsrc.p, g.data(), g.size() * sizeof(long long), cudaMemcpyHostToDevice, stream));
    d.cfac.alloc(g.size());
    d.prow_off.alloc(d.xoff.size());
    CK(cudaMemcpyAsync(d.prow_off.p, d.xoff.data(), d.xoff.size() * sizeof(int), cudaMemcpyHostToDevice, stream));
    d.prow_node.alloc(pnode.size());
    CK(cudaMemcpyAsync(d.prow_node.p, pnode.data(), pnode.size() * sizeof(int), cudaMemcpyHostToDevice, stream));
    d.prow_phase.alloc(pphase.size());
    CK(cudaMemcpyAsync(d.prow_phase.p, pphase.data(), pphase.size(), cudaMemcpyHostToDevice, stream));
    // cfac starts at a 16-byte boundary after x; the int program after cfac
    const size_t xb = size_t(P.nphi) * sizeof(double2);
    const size_t all = xb + size_t(P.ncf) * sizeof(double2) + size_t(P.nmeta) * sizeof(int);
    if (xb > size_t(optin_smem)) throw Error("solution vector does not fit in shared memory");
    d.smem_factor = all <= size_t(optin_smem) ? 1 : 0;
    d.smem_bytes = int(d.smem_factor ? all : xb);
    // warp-per-rhs layout: staged factor + W solution vectors
    const size_t fac = size_t(P.ncf) * sizeof(double2) + size_t(P.nmeta) * sizeof(int);
    d.wsm_factor = 0;
    d.wwarps = 0;
    for (int w = 8; w >= 1; w /= 2)
      if (fac + size_t(w) * xb <= size_t(optin_smem)) {
        d.wsm_factor = 1;
        d.wwarps = w;
        break;
      }
    if (!d.wsm_factor)
      for (int w = 8; w >= 1; w /= 2)
        if (size_t(w) * xb <= size_t(optin_smem)) {
          d.wwarps = w;
          break;
        }
    d.wsmem_bytes = int((d.wsm_factor ? fac : 0) + size_t(std::max(d.wwarps, 1)) * xb);
    CK(cudaStreamSynchronize(stream));
  }

  template <int MODE>
  void launch_csolve(DevElim& d, const CSolveArgs& c, int nrhs) {
    if (nrhs <= 0) return;
    if (d.wwarps > 0) {
      const int W = d.wwarps;
      const unsigned grid = unsigned((nrhs + W - 1) / W);
      if (d.wsm_factor)
        csolve_warp_kernel<MODE, true><<<grid, 32 * W, d.wsmem_bytes, stream>>>(c, nrhs);
      else
        csolve_warp_kernel<MODE, false><<<grid, 32 * W, d.wsmem_bytes, stream>>>(c, nrhs);
    } else {
      csolve_kernel<MODE><<<nrhs, 256, d.smem_bytes, stream>>>(c);
    }
    launched();
    CK(cudaGetLastError());
  }

  // K1f on the device: blocks <- input, fill <- 0, then the level executor,
  // then the present-phase compaction of the factor.
  // check_now=false defers the singular-pivot check to check_deferred_fail()
  // (no host round trip inside a run; the run's final sync reads the flag)
  void factorize(DevElim& d, const double2* d_input, double floor, bool check_now = true) {
    const ElimSchedule& h = d.h;
    if (h.n_input > 0)
      CK(cudaMemcpyAsync(d.blocks.p, d_input, size_t(h.n_input) * 9 * sizeof(double2), cudaMemcpyDeviceToDevice,
                         stream));
    if (h.nblocks > h.n_input)
      CK(cudaMemsetAsync(d.blocks.p + size_t(h.n_input) * 9, 0, size_t(h.nblocks - h.n_input) * 9 * sizeof(double2),
                         stream));
    CK(cudaMemsetAsync(d.fail.p, 0xff, sizeof(unsigned long long), stream));
    if (h.nlevels > 0) {
      ElimDev e;
      e.nlevels = h.nlevels;
      e.step_node = d.P(A_STEP_NODE);
      e.step_diag = d.P(A_STEP_DIAG);
      e.lvl_step_off = d.P(A_LVL_STEP_OFF);
      e.lvl_steps = d.P(A_LVL_STEPS);
      e.lvl_slot_off = d.P(A_LVL_SLOT_OFF);
      e.lvl_slots = d.P(A_LVL_SLOTS);
      e.lvl_slot_step = d.P(A_LVL_SLOT_STEP);
      e.slot_from = d.P(A_SLOT_FROM);
      e.slot_to = d.P(A_SLOT_TO);
      e.lvl_apply_off = d.P(A_LVL_APPLY_OFF);
      e.apply_blk = d.P(A_APPLY_BLK);
      e.apply_off = d.P(A_APPLY_OFF);
      e.apply_slots = d.P(A_APPLY_SLOTS);
      e.mask = d.mask.p;
      e.blocks = d.blocks.p;
      e.pinv = d.pinv.p;
      e.contrib = d.contrib.p;
      e.pivot_floor = floor;
      e.fail = d.fail.p;
      e.fail_pivot = d.fail_pivot.p;
      elim_factor_kernel<<<1, ELIM_THREADS, 0, stream>>>(e);
      launched();
      CK(cudaGetLastError());
    }
    if (!check_now) {
      CK(cudaMemcpyAsync(h_fail, d.fail.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
      deferred_fail = &d;
    } else {
      unsigned long long failed = 0;
      CK(cudaMemcpyAsync(&failed, d.fail.p, sizeof(failed), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      throw_if_failed(d, failed);
    }
    if (d.ncf_all > 0) {
      compact_gather_kernel<<<(d.ncf_all + 255) / 256, 256, 0, stream>>>(d.ncf_all, d.gsrc.p, d.blocks.p,
                                                                         d.pinv.p, d.cfac.p);
      launched();
      CK(cudaGetLastError());
    }
  }

  unsigned long long* h_fail = nullptr;  // pinned
  DevElim* deferred_fail = nullptr;
  // after a stream sync: raise the SolverError a deferred factorization recorded
  void check_deferred_fail() {
    if (!deferred_fail) return;
    DevElim* d = deferred_fail;
    deferred_fail = nullptr;
    throw_if_failed(*d, *h_fail);
  }

  void throw_if_failed(DevElim& d, unsigned long long failed) {
    const ElimSchedule& h = d.h;
    if (failed != ~0ull) {
      double piv = 0;
      CK(cudaMemcpy(&piv, d.fail_pivot.p + failed, sizeof(double), cudaMemcpyDeviceToHost));
      const int node = h.step_node[size_t(failed)];
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.3e", piv);
      throw SolverError("singular present-phase diagonal while eliminating node " + std::to_string(node) +
                            " (smallest pivot " + buf + ", " + std::to_string(h.nsteps - int(failed)) + " of " +
                            std::to_string(h.nsteps) + " eliminations left)",
                        piv, node);
    }
  }

  CSolveArgs cargs(DevElim& d, const double2* kept_val) {
    CSolveArgs a{};
    a.P = d.prog;
    a.meta_g = d.meta.p;
    a.cfac_g = d.cfac.p;
    a.kept_val = kept_val;
    a.smem_factor = d.smem_factor;
    a.n = d.h.n;
    a.prow_off = d.prow_off.p;
    a.mask = d.mask.p;
    a.prow_node = d.prow_node.p;
    a.prow_phase = d.prow_phase.p;
    return a;
  }

  // anchored solves: rhs [nrhs][3n] (device, may be null = zero) -> out [nrhs][3n]
  void solve_full(DevElim& d, const double2* kept_val, const double2* rhs, int nrhs, double2* out) {
    if (nrhs <= 0) return;
    CSolveArgs a = cargs(d, kept_val);
    a.rhs_full = rhs;
    a.out_full = out;
    launch_csolve<CM_FULL>(d, a, nrhs);
  }

  // refresh_base (reduce.cpp:265-268): base = solve(i_agg) for every scenario
  long long* dbg_clock = nullptr;
  // s, r >= 0: the commit that changed i_agg (incremental forward walk)
  void refresh_base(int s = -1, int r = -1) {
    if (full.bW > 0) {
      BaseArgs b = full.bprog;
      b.L = L;
      b.W = full.bW;
      b.cfac = full.cfac.p;
      b.meta = full.bmeta.p;
      b.iaggp = d_iaggp.p;
      b.kept_val = d_slackv.p;
      b.bv = d_bv.p;
      b.dbg = dbg_clock;
      b.tfwd = b.walk >= 0 ? d_tfwd.p : nullptr;
      b.inc = (b.walk >= 0 && s >= 0 && !force_full_refresh) ? 1 : 0;
      b.inc_s = s;
      b.inc_r = r;
      if (profile) CK(cudaEventRecord(ev_a, stream));
      if (full.bsm)
        base_refresh_kernel<true><<<(L + b.W - 1) / b.W, 32 * b.W * b.WB, full.bsmem, stream>>>(b);
      else
        base_refresh_kernel<false><<<(L + b.W - 1) / b.W, 32 * b.W * b.WB, full.bsmem, stream>>>(b);
      launched();
      CK(cudaGetLastError());
      if (profile) {
        const float ms = event_ms();
        solve_stats.launches += 1;
        solve_stats.ms += ms;
        solve_stats.flops += double(L) * double(full.prog.ncf) * 8.0;
        solve_stats.bytes += double(full.prog.ncf) * 16.0 + double(L) * double(nphi) * 16.0 * 2.0;
      }
      return;
    }
    CSolveArgs c = cargs(full, d_slackv.p);
    c.dbg = dbg_clock;
    c.iagg = d_iagg.p;
    c.base = d_bv.p;
    c.L = L;
    if (profile) CK(cudaEventRecord(ev_a, stream));
    launch_csolve<CM_BASE>(full, c, L);
    if (profile) {
      const float ms = event_ms();
      solve_stats.launches += 1;
      solve_stats.ms += ms;
      solve_stats.flops += double(L) * double(full.prog.ncf) * 8.0;
      solve_stats.bytes += double(full.prog.ncf) * 16.0 + double(L) * double(nphi) * 16.0 * 2.0;
    }
  }

  // Z columns solve(e_k) - v0 at present rows (reduce.cpp:272-290)
  void build_z() {
    d_Z.alloc(size_t(nphi) * size_t(nphi));
    CSolveArgs c = cargs(full, d_slackv.p);
    c.col0 = 0;
    c.v0p = d_v0p.p;
    c.zout = d_Z.p;
    launch_csolve<CM_ZCOL>(full, c, nphi);
  }

  Impl(const Problem& p, int dev_id) : prob(p), device(dev_id) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw CudaError("no CUDA device available (the B200 path has no CPU fallback)");
    if (device < 0) CK(cudaGetDevice(&device));
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CK(cudaMallocHost(&h_fail, sizeof(unsigned long long)));
    CK(cudaDeviceGetAttribute(&optin_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    parse_s1_gk();
    for (auto fn : {csolve_kernel<CM_FULL>, csolve_kernel<CM_BASE>, csolve_kernel<CM_ZCOL>})
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin_smem));
    for (auto fn : {csolve_warp_kernel<CM_FULL, true>, csolve_warp_kernel<CM_BASE, true>,
                    csolve_warp_kernel<CM_ZCOL, true>, csolve_warp_kernel<CM_FULL, false>,
                    csolve_warp_kernel<CM_BASE, false>, csolve_warp_kernel<CM_ZCOL, false>})
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin_smem));
    for (auto fn : {score_kernel<false>, score_kernel<true>})
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin_smem));
    CK(cudaFuncSetAttribute(score3_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin_smem - 256));
    CK(cudaFuncSetAttribute(score3_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin_smem - 256));
    CK(cudaFuncSetAttribute(base_refresh_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin_smem - 64));
    CK(cudaFuncSetAttribute(base_refresh_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin_smem - 64));
    CK(cudaFuncSetAttribute(naive_score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin_smem - 64));
    CK(cudaFuncSetAttribute(naive_score_global_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin_smem - 64));
    n = prob.y.n;
    prow_off.assign(size_t(n) + 1, 0);
    for (int i = 0; i < n; ++i) {
      const PhaseMask m{prob.mask[size_t(i)]};
      prow_off[size_t(i) + 1] = prow_off[size_t(i)] + m.count();
      for (int ph = 0; ph < 3; ++ph)
        if (m.has(ph)) {
          prow_node.push_back(i);
          prow_phase.push_back(std::uint8_t(ph));
        }
    }
    nphi = prow_off[size_t(n)];
    d_prow_off.alloc(prow_off.size());
    CK(cudaMemcpy(d_prow_off.p, prow_off.data(), prow_off.size() * sizeof(int), cudaMemcpyHostToDevice));
    d_prow_node.alloc(prow_node.size());
    d_prow_phase.alloc(prow_phase.size());
    if (nphi > 0) {
      CK(cudaMemcpy(d_prow_node.p, prow_node.data(), prow_node.size() * sizeof(int), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(d_prow_phase.p, prow_phase.data(), prow_phase.size(), cudaMemcpyHostToDevice));
    }
    d_mask.alloc(size_t(n));
    CK(cudaMemcpy(d_mask.p, prob.mask.data(), size_t(n), cudaMemcpyHostToDevice));
    d_yin.alloc(prob.y.row.size() * 9);
    if (!prob.y.row.empty())
      CK(cudaMemcpy(d_yin.p, prob.y.val.data(), prob.y.val.size() * sizeof(double), cudaMemcpyHostToDevice));
    pivot_floor = 1e-12 * std::max(prob.y.max_abs(), 1.0);
    if (prob.slack < 0) return;  // matrix-only engine (kron_reduce on a bare Y)
    std::vector<int> elim;
    for (int i = 0; i < n; ++i)
      if (i != prob.slack) elim.push_back(i);
    upload_elim(full, prob.y, prob.mask, elim);
    double sv[6];
    for (int q = 0; q < 3; ++q) {
      sv[2 * q] = prob.net.nodes[size_t(prob.slack)].slack_voltage[q].real();
      sv[2 * q + 1] = prob.net.nodes[size_t(prob.slack)].slack_voltage[q].imag();
    }
    d_slackv.alloc(3);
    CK(cudaMemcpy(d_slackv.p, sv, sizeof sv, cudaMemcpyHostToDevice));
    // the anchored factorization every solve of this engine uses (solver.cpp:168-179)
    factorize(full, d_yin.p, pivot_floor);
    d_v0.alloc(size_t(3) * n);
    d_v0p.alloc(size_t(std::max(nphi, 1)));
    d_cand.alloc(size_t(2 * n));
    // candidate lists: sized once for both the host-fed (2n) and the device
    // loop (2 nb + 1) paths, never reallocated (the loop graph captures them)
    d_cs.alloc(size_t(2 * std::max(n, int(prob.net.branches.size()))) + 1);
    d_cr.alloc(size_t(2 * std::max(n, int(prob.net.branches.size()))) + 1);
    d_snt.alloc(size_t(n));
    d_snid.alloc(size_t(n));
    d_memoff.alloc(size_t(n) + 1);
    d_memlist.alloc(size_t(n));
    CK(cudaMallocHost(&h_cand, sizeof(int4) * size_t(2 * n)));
    CK(cudaMallocHost(&h_snt, sizeof(unsigned) * size_t(n)));
    d_tab.alloc(size_t(4) * n + size_t(nphi) + kTabPad);
    d_tplain.alloc((size_t(4) * n + size_t(nphi) + kTabPad) / 16 + 2);
    d_cidx.alloc(size_t(2 * n));
    CK(cudaMallocHost(&h_tab, sizeof(unsigned) * (size_t(4) * n + size_t(nphi) + kTabPad)));
    CK(cudaMallocHost(&h_cidx, sizeof(int) * size_t(2 * n)));
    tab_of_node.assign(size_t(n), -1);
    sn_pos.assign(size_t(n), -1);
    if (prob.L > 0) load_scenarios(prob.scenario_ids, prob.injections, prob.voltages);
  }

  // ScenarioLibrary on the device (load_library: V-hat = solve(I-hat) when
  // the voltages are not given, scenario.cpp:39-50).
  // Host <-> device copies of the per-call inputs and results (reload, the
  // scenario library) through one pinned staging buffer kept by the engine:
  // a memcpy into pinned memory plus an async DMA beats a pageable copy
  // (driver bounce buffers) for these 0.1-2 MB transfers.
  char* h_stage = nullptr;
  size_t h_stage_cap = 0;
  char* stage_buf(size_t bytes) {
    if (h_stage_cap < bytes) {
      if (h_stage) CK(cudaFreeHost(h_stage));
      h_stage = nullptr;
      CK(cudaMallocHost(reinterpret_cast<void**>(&h_stage), bytes));
      h_stage_cap = bytes;
    }
    return h_stage;
  }
  void h2d_staged(void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    char* p = stage_buf(bytes);
    CK(cudaStreamSynchronize(stream));  // the buffer's previous transfer is done
    std::memcpy(p, src, bytes);
    CK(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, stream));
  }
  void d2h_staged(void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    char* p = stage_buf(bytes);
    CK(cudaMemcpyAsync(p, src, bytes, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    std::memcpy(dst, p, bytes);
  }

  void load_scenarios(const std::vector<std::string>& ids, const std::vector<double>& inj,
                      const std::vector<double>& volt) {
    if (comm && (24 + 8 * int(ids.size()) + 15) / 16 * 16 > rec_bytes)
      throw ConfigError("set_comm before loading a library with more scenarios (exchange records are sized by L)");
    L = int(ids.size());
    prob.L = L;
    prob.scenario_ids = ids;
    prob.injections = inj;
    if (L == 0) return;
    d_inj.alloc(size_t(L) * 3 * n);
    h2d_staged(d_inj.p, inj.data(), inj.size() * sizeof(double));
    d_vhat.alloc(size_t(L) * 3 * n);
    if (!volt.empty()) {
      CK(cudaStreamSynchronize(stream));  // (one staging buffer)
      CK(cudaMemcpy(d_vhat.p, volt.data(), volt.size() * sizeof(double), cudaMemcpyHostToDevice));
      h_vhat = volt;
    } else {
      solve_full(full, d_slackv.p, d_inj.p, L, d_vhat.p);
      h_vhat.resize(size_t(L) * 6 * n);
      d2h_staged(h_vhat.data(), d_vhat.p, h_vhat.size() * sizeof(double));
    }
    prob.voltages.clear();  // (volt may alias it) V-hat lives in h_vhat (Engine::vhat)
    d_vhatp.alloc(size_t(nphi) * L);
    d_bv.alloc(size_t(nphi) * L * 2);
    d_iagg.alloc(size_t(n) * L * 3);
    d_iaggp.alloc(size_t(L) * std::max(nphi, 1));
    d_tfwd.alloc(size_t(L) * std::max(nphi, 1));
    d_psmice.alloc(size_t(s3_ldc()) * L);
    d_pmaxerr.alloc(size_t(s3_ldc()) * L);
    d_grpdone.alloc(s3_groups_max());
    CK(cudaMemset(d_grpdone.p, 0, d_grpdone.n * sizeof(int)));
    d_pcand.alloc(size_t(2 * n));
    d_best.alloc(size_t(2 + L));
    if (!h_best || h_best_n < size_t(2 + L)) {  // pinned readback slot, kept across reloads
      if (h_best) cudaFreeHost(h_best);
      CK(cudaMallocHost(&h_best, sizeof(double) * size_t(2 + L)));
      h_best_n = size_t(2 + L);
    }
  }

  ~Impl() {
    free_comm();
    if (ev_a) {
      cudaEventDestroy(ev_a);
      cudaEventDestroy(ev_b);
      cudaEventDestroy(ev_run0);
      cudaEventDestroy(ev_run1);
    }
    if (h_best) cudaFreeHost(h_best);
    if (h_stage) cudaFreeHost(h_stage);
    if (h_fail) cudaFreeHost(h_fail);
    if (h_loopst) cudaFreeHost(h_loopst);
    if (h_trace) cudaFreeHost(h_trace);
    if (h_live) cudaFreeHost(h_live);
    if (h_cand) cudaFreeHost(h_cand);
    if (h_snt) cudaFreeHost(h_snt);
    if (h_tab) cudaFreeHost(h_tab);
    if (h_cidx) cudaFreeHost(h_cidx);
    if (loop_exec) cudaGraphExecDestroy(loop_exec);
    if (loop_graph) cudaGraphDestroy(loop_graph);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (stream2) cudaStreamDestroy(stream2);
    if (stream3) cudaStreamDestroy(stream3);
    if (stream_cap) cudaStreamDestroy(stream_cap);
    if (ev_fork3) cudaEventDestroy(ev_fork3);
    if (ev_join3) cudaEventDestroy(ev_join3);
    if (stream) cudaStreamDestroy(stream);
  }

  // ---- loop --------------------------------------------------------------
  void begin(const ReductionConfig& c) {
    if (!(c.e_bar >= 0)) throw ConfigError("e_bar must be non-negative");
    if (c.target_reduction && !(*c.target_reduction >= 0 && *c.target_reduction <= 1))
      throw ConfigError("target_reduction must lie in [0,1]");
    if (L == 0) throw ValidationError("scenario library is empty");
    if (!c.use_delta && full.bW <= 0)
      throw ConfigError("use_delta=false: the solution vector does not fit in shared memory");
    cfg = c;
    // AnchoredSolver (re-factorized per run, as run_reduction does, reduce.cpp:359)
    factorize(full, d_yin.p, pivot_floor, /*check_now=*/false);
    solve_full(full, d_slackv.p, nullptr, 1, d_v0.p);
    if (nphi > 0) {
      gather_rows_kernel<<<(nphi + 255) / 256, 256, 0, stream>>>(nphi, d_prow_node.p, d_prow_phase.p, d_v0.p, d_v0p.p);
      launched();
      CK(cudaGetLastError());
    }
    const int tot = std::max(nphi * L, n * L * 3);
    prep_kernel<<<(tot + 255) / 256, 256, 0, stream>>>(n, L, nphi, d_prow_node.p, d_prow_phase.p, d_vhat.p, d_inj.p,
                                                       d_vhatp.p, d_bv.p, d_iagg.p, d_iaggp.p);
    launched();
    CK(cudaGetLastError());
    build_z();
    refresh_base();
    hs.init(prob.net, &prob.injections, L);
    loop_active = true;
  }

  bool target_reached() const { return cfg.target_reduction && hs.reduction_fraction() >= *cfg.target_reduction; }

  // per-iteration inputs: super-node table + candidates (pinned, async)
  void upload_iteration(long long c0, long long c1) {
    const long long C = c1 - c0;
    if (!cfg.use_delta) {
      // full-solve path: candidate lists + super-node / member CSR
      if (C > 0) {
        CK(cudaMemcpyAsync(d_cs.p, cs.data() + c0, size_t(C) * sizeof(int), cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(d_cr.p, cr.data() + c0, size_t(C) * sizeof(int), cudaMemcpyHostToDevice, stream));
      }
      upload_members();
      return;
    }
    if (cfg.objective == Objective::magnitude) {
      // 4-row blocks that never split a super-node; inert padding rows
      // (phase field 3) fill each block
      constexpr unsigned kPad = 7u;  // rho 0, first, phase 3
      int t = 0;
      for (int i : hs.supernodes) {
        const unsigned m = prob.mask[size_t(i)];
        const int rows = __builtin_popcount(m);
        if ((t & 3) + rows > 4)
          while (t & 3) h_tab[t++] = kPad;
        tab_of_node[size_t(i)] = t;
        unsigned first = 4u;
        for (int p = 0; p < 3; ++p)
          if ((m >> p) & 1u) {
            const unsigned rho = unsigned(prow_off[size_t(i)] + __builtin_popcount(m & ((1u << p) - 1u)));
            h_tab[t++] = (rho << 3) | first | unsigned(p);
            first = 0u;
          }
      }
      while (t & 3) h_tab[t++] = kPad;
      R = t;
      for (int u = 0; u < kTabPad; ++u) h_tab[R + u] = kPad;
      int cnt[4] = {0, 0, 0, 0};
      for (long long c = c0; c < c1; ++c) ++cnt[__builtin_popcount(prob.mask[size_t(cr[size_t(c)])])];
      grp_off[0] = 0;
      grp_off[1] = cnt[1];
      grp_off[2] = cnt[1] + cnt[2];
      grp_off[3] = cnt[1] + cnt[2] + cnt[3];
      int fill[4] = {0, 0, grp_off[1], grp_off[2]};
      for (long long c = c0; c < c1; ++c) {
        const int s = cs[size_t(c)], r = cr[size_t(c)];
        const int g = __builtin_popcount(prob.mask[size_t(r)]);
        const int pos = fill[g]++;
        h_cand[pos] = make_int4(s, r, tab_of_node[size_t(s)], tab_of_node[size_t(r)]);
        h_cidx[pos] = int(c - c0);
      }
      if (C > 0) {
        CK(cudaMemcpyAsync(d_cand.p, h_cand, size_t(C) * sizeof(int4), cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(d_cidx.p, h_cidx, size_t(C) * sizeof(int), cudaMemcpyHostToDevice, stream));
      }
      CK(cudaMemcpyAsync(d_tab.p, h_tab, size_t(R + kTabPad) * sizeof(unsigned), cudaMemcpyHostToDevice, stream));
      {
        const int ntiles = (R + 15) / 16;
        h_tplain.assign(size_t(ntiles) + 1, 0);
        for (int t = 0; t < ntiles; ++t) {
          unsigned all = 0xffffffffu, pad = 0u;
          for (int u = 0; u < 16; ++u) {
            const unsigned e = h_tab[16 * t + u];
            all &= e;
            pad |= e & (e >> 1) & 1u;
          }
          h_tplain[size_t(t)] = (all & 4u) && !pad ? 1 : 0;
        }
        CK(cudaMemcpyAsync(d_tplain.p, h_tplain.data(), h_tplain.size(), cudaMemcpyHostToDevice, stream));
      }
      return;
    }
    int k = 0;
    for (int i : hs.supernodes) {
      sn_pos[size_t(i)] = k;
      h_snt[k++] = (unsigned(prow_off[size_t(i)]) << 3) | unsigned(prob.mask[size_t(i)]);
    }
    for (long long c = c0; c < c1; ++c) {
      const int s = cs[size_t(c)], r = cr[size_t(c)];
      h_cand[c - c0] = make_int4(s, r, sn_pos[size_t(s)], sn_pos[size_t(r)]);
    }
    if (C > 0) CK(cudaMemcpyAsync(d_cand.p, h_cand, size_t(C) * sizeof(int4), cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_snt.p, h_snt, size_t(k) * sizeof(unsigned), cudaMemcpyHostToDevice, stream));
    if (cfg.objective == Objective::complex_error) upload_members();
  }

  // members of every super-node (CSR by id) and the ascending super-node list
  void upload_members() {
    std::vector<int> off(size_t(n) + 1, 0), lst;
    for (int i = 0; i < n; ++i) {
      for (int j : hs.members[size_t(i)]) lst.push_back(j);
      off[size_t(i) + 1] = int(lst.size());
    }
    CK(cudaMemcpy(d_memoff.p, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice));
    if (!lst.empty()) CK(cudaMemcpy(d_memlist.p, lst.data(), lst.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_snid.p, hs.supernodes.data(), hs.supernodes.size() * sizeof(int), cudaMemcpyHostToDevice));
  }

  // use_delta=false scorer (kernels_naive.cuh): one warp per (candidate, scenario)
  void launch_naive(long long C) {
    BaseArgs b = full.bprog;
    b.L = L;
    b.cfac = full.cfac.p;
    b.meta = full.bmeta.p;
    b.iaggp = d_iaggp.p;
    b.kept_val = d_slackv.p;
    const size_t fixed = size_t(b.ncf) * 16 + size_t(b.nmeta) * 4;
    const size_t per_warp = size_t(nphi) * 16 + size_t(n) * 8;
    int W = 0;
    for (int w = 8; w >= 1; --w)
      if (fixed + size_t(w) * per_warp <= size_t(optin_smem) - 64) {
        W = w;
        break;
      }
    if (W == 0 || !full.bsm || std::getenv("KRONRED_NAIVE_GLOBAL")) {
      // program too large for shared memory: read it from global memory, one
      // pair per CTA of WB warps (the layout of the global refresh program)
      NaiveArgs q{};
      b.W = 1;
      q.b = b;
      q.C = int(C);
      q.cs = d_cs.p;
      q.cr = d_cr.p;
      q.ns = int(hs.supernodes.size());
      q.sn_id = d_snid.p;
      q.mem_off = d_memoff.p;
      q.mem_list = d_memlist.p;
      q.mask = d_mask.p;
      q.prow_off = d_prow_off.p;
      q.vhat_full = d_vhat.p;
      q.n = n;
      q.e_bar = cfg.e_bar;
      q.complex_obj = cfg.objective == Objective::complex_error ? 1 : 0;
      q.out_sm = d_psmice.p;
      q.out_mx = d_pmaxerr.p;
      q.ldc = s3_ldc();
      const size_t sm = size_t(nphi) * 16 + size_t(n) * 8;
      if (sm > size_t(optin_smem) - 64) throw ConfigError("use_delta=false: the solution vector does not fit in shared memory");
      int sms = 0;
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
      const long long pairs = C * L;
      const int grid = int(std::max<long long>(1, std::min<long long>(pairs, 2LL * sms)));
      naive_score_global_kernel<<<grid, 32 * std::max(1, b.WB), sm, stream>>>(q);
      launched();
      CK(cudaGetLastError());
      return;
    }
    b.W = W;
    NaiveArgs q{};
    q.b = b;
    q.C = int(C);
    q.cs = d_cs.p;
    q.cr = d_cr.p;
    q.ns = int(hs.supernodes.size());
    q.sn_id = d_snid.p;
    q.mem_off = d_memoff.p;
    q.mem_list = d_memlist.p;
    q.mask = d_mask.p;
    q.prow_off = d_prow_off.p;
    q.vhat_full = d_vhat.p;
    q.n = n;
    q.e_bar = cfg.e_bar;
    q.complex_obj = cfg.objective == Objective::complex_error ? 1 : 0;
    q.out_sm = d_psmice.p;
    q.out_mx = d_pmaxerr.p;
    q.ldc = s3_ldc();
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const long long pairs = C * L;
    const int grid = int(std::max<long long>(1, std::min<long long>((pairs + W - 1) / W, 4LL * sms)));
    naive_score_kernel<<<grid, 32 * W, fixed + size_t(W) * per_warp, stream>>>(q);
    launched();
    CK(cudaGetLastError());
  }

  void launch_score(long long C) {
    if (C <= 0) return;
    if (profile) CK(cudaEventRecord(ev_a, stream));
    if (!cfg.use_delta) {
      launch_naive(C);
    } else if (cfg.objective == Objective::magnitude) {
      // score3 (kernels_score3.cuh): work items = candidate group x scenario slice
      S3Args q = s3_args();
      q.C = int(C);
      q.R = R;
      q.S = s3_lanes(C * L, s3_fill(), s3_force, s3_fill4_16());
      int c3 = 0;
      for (int k = 1; k <= 3; ++k) {
        const int cpc = !s1_ok() ? s3_cpc(s3_slots(), k, q.S)
                                 : (k == 1 ? s1_gk[s1_switch_index(q.S)] : s3_cpc(s3_slots(), k, q.s_multi));
        q.grp_start[k] = grp_off[k - 1];
        q.grp_cta[k - 1] = c3;
        c3 += (grp_off[k] - grp_off[k - 1] + cpc - 1) / cpc * q.nsl;
      }
      q.grp_cta[3] = c3;
      if (s1_ok()) {
        launch_s1(q.S, q, q.grp_cta[1], stream);
        if (profile) {  // score1 timed on its own (the roofline kernel); score3's share below
          const float ms = event_ms();
          double f, b;
          score_work(score_c0, score_c0 + C, f, b, 1);
          score_stats.launches += 1;
          score_stats.ms += ms;
          score_stats.flops += f;
          score_stats.bytes += b;
          CK(cudaEventRecord(ev_a, stream));
        }
        q.skip_nl1 = 1;
        if (c3 > q.grp_cta[1]) {
          score3_kernel<0><<<c3 - q.grp_cta[1], s3_threads(), S3Layout{s3_ls(), s3_slots()}.smem_bytes(), stream>>>(q);
          launched();
          CK(cudaGetLastError());
        }
        if (profile) {
          const float ms = event_ms();
          double f, b;
          score_work(score_c0, score_c0 + C, f, b, 2);
          multi_stats.launches += c3 > q.grp_cta[1] ? 1 : 0;
          multi_stats.ms += ms;
          multi_stats.flops += f;
          multi_stats.bytes += b;
        }
        return;
      } else if (c3 > 0) {
        if (q.S == 1)
          score3_kernel<1><<<c3, s3_threads(), S3Layout{s3_ls(), s3_slots()}.smem_bytes(), stream>>>(q);
        else  // the split program stages G / S slots in its own ring
          score3_kernel<0><<<c3, s3_threads(), S3Layout{s3_ls(), s3_slots(), q.S, S3_NS_SPLIT}.smem_bytes(), stream>>>(q);
        launched();
        CK(cudaGetLastError());
      }
    } else {
      launch_score_members(C);
    }
    if (profile) {
      const float ms = event_ms();
      double f, b;
      score_work(score_c0, score_c0 + C, f, b);
      score_stats.launches += 1;
      score_stats.ms += ms;
      score_stats.flops += f;
      score_stats.bytes += b;
    }
  }

  // complex-objective scorer geometry and buffers for C candidates
  ScoreArgs members_args(long long C) {
    ScoreArgs a{};
    a.C = int(C);
    a.L = L;
    a.nphi = nphi;
    a.ns = int(hs.supernodes.size());
    int P = L * (32 / gcd_int(L, 32));
    if (P > 512) P = L;
    a.G = P / L;
    const long long ctas = (C + a.G - 1) / a.G;
    const int smax = std::max(1, 512 / P);
    const long long want = (148LL * 1536 + ctas * P - 1) / (ctas * P);
    a.S = int(std::min<long long>(smax, std::max<long long>(1, want)));
    a.K = 64;
    a.cand = d_cand.p;
    a.snt = d_snt.p;
    a.mask = d_mask.p;
    a.prow_off = d_prow_off.p;
    a.Z = d_Z.p;
    a.bv = d_bv.p;
    a.iagg = d_iagg.p;
    a.mem_off = d_memoff.p;
    a.mem_list = d_memlist.p;
    a.sn_id = d_sn.p;
    a.vhatp = d_vhatp.p;
    a.out_smice = d_psmice.p;
    a.out_maxerr = d_pmaxerr.p;
    return a;
  }

  void launch_score_members(long long C) {
    ScoreArgs a{};
    a.C = int(C);
    a.L = L;
    a.nphi = nphi;
    a.ns = int(hs.supernodes.size());
    // pairs per CTA: a multiple of 32 so each warp shares one segment
    int P = L * (32 / gcd_int(L, 32));
    if (P > 512) P = L;
    a.G = P / L;
    const long long ctas = (C + a.G - 1) / a.G;
    const int smax = std::max(1, 512 / P);
    const long long want = (148LL * 1536 + ctas * P - 1) / (ctas * P);
    a.S = int(std::min<long long>(smax, std::max<long long>(1, want)));
    a.K = 64;
    const size_t smem = size_t(std::max(a.K, a.S)) * size_t(P) * sizeof(double);
    a.cand = d_cand.p;
    a.snt = d_snt.p;
    a.mask = d_mask.p;
    a.prow_off = d_prow_off.p;
    a.Z = d_Z.p;
    a.bv = d_bv.p;
    a.iagg = d_iagg.p;
    a.mem_off = d_memoff.p;
    a.mem_list = d_memlist.p;
    a.sn_id = d_snid.p;
    a.vhatp = d_vhatp.p;
    a.out_smice = d_psmice.p;
    a.out_maxerr = d_pmaxerr.p;
    if (cfg.objective == Objective::complex_error)
      score_kernel<true><<<unsigned(ctas), P * a.S, smem, stream>>>(a);
    else
      score_kernel<false><<<unsigned(ctas), P * a.S, smem, stream>>>(a);
    launched();
    CK(cudaGetLastError());
  }

  // score [c0,c1) and reduce to the local best: (smice, global idx, max_err) in h_best
  void score_best(long long c0, long long c1) {
    const long long C = c1 - c0;
    score_c0 = c0;
    upload_iteration(c0, c1);
    launch_score(C);
    const bool naive = !cfg.use_delta;
    argmin_kernel<<<1, 1024, 0, stream>>>(int(std::max(C, 0LL)), L,
                                          (naive || cfg.objective == Objective::magnitude) ? s3_ldc() : 0,
                                          cfg.e_bar, c0, d_psmice.p, d_pmaxerr.p,
                                          (cfg.objective == Objective::magnitude && !naive) ? d_pcand.p : nullptr,
                                          d_best.p);
    launched();
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h_best, d_best.p, sizeof(double) * size_t(2 + L), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
  }

  long long best_index() const {
    long long idx;
    std::memcpy(&idx, &h_best[1], sizeof idx);
    return idx;
  }

  // multi-GPU min-loc over ranks (lexicographic (smice, idx))
  void exchange_best() {
    if (world <= 1 || xfn == nullptr) return;
    const size_t bytes = sizeof(double) * size_t(2 + L);
    std::vector<double> all(size_t(world) * size_t(2 + L));
    if (xfn(xuser, h_best, all.data(), bytes) != 0) throw Error("exchange callback failed");
    int bw = -1;
    double bs = 0;
    long long bi = -1;
    for (int w = 0; w < world; ++w) {
      const double* rec = all.data() + size_t(w) * size_t(2 + L);
      long long idx;
      std::memcpy(&idx, &rec[1], sizeof idx);
      if (idx < 0) continue;
      if (bi < 0 || rec[0] < bs || (rec[0] == bs && idx < bi)) {
        bs = rec[0];
        bi = idx;
        bw = w;
      }
    }
    if (bw >= 0) {
      std::memcpy(h_best, all.data() + size_t(bw) * size_t(2 + L), bytes);
    } else {
      const long long none = -1;
      std::memcpy(&h_best[1], &none, sizeof none);
    }
  }

  // ---- device-resident loop ------------------------------------------------
  static size_t pow2_at_least(size_t x) {
    size_t p = 1;
    while (p < x) p <<= 1;
    return p;
  }
  // enumeration keys: a power-of-two sort region, then the previous sorted list
  size_t enum_kcap() const { return pow2_at_least(std::max<size_t>(2 * prob.net.branches.size(), 1)); }
  size_t enum_smem() const { return (enum_kcap() + 2 * prob.net.branches.size() + 1) * sizeof(unsigned); }

  bool device_loop_ok(const ReductionConfig& c) const {
    return !force_host_loop && c.use_delta && (world == 1 || comm) && !profile &&
           full.bW > 0 && n <= 65535 && enum_smem() + 24 * 1024 <= size_t(optin_smem);
  }

  LoopArgs loop_args() {
    LoopArgs a{};
    a.st = d_loopst.p;
    a.n = n;
    a.nb = int(prob.net.branches.size());
    a.slack = prob.slack;
    a.L = L;
    a.nphi = nphi;
    a.cap = n;
    a.e_bar = cfg.e_bar;
    a.kcap = int(enum_kcap());
    a.inc_enum = std::getenv("KRONRED_ENUM_FULL") == nullptr ? 1 : 0;
    a.nsl = s3_nsl();
    a.G3 = s3_slots();
    for (int i = 0; i < 3; ++i) a.gk1[i] = s1_ok() ? s1_gk[i] : 0;
    a.s_multi = s3_multi_lanes();
    a.fill = s3_fill();
    a.fill4_16 = s3_fill4_16();
    a.force_s = s3_force;
    a.ldc = s3_ldc();  // max_err is scenario-major; per-candidate SMICE in pcand
    a.complex_obj = cfg.objective == Objective::complex_error ? 1 : 0;
    a.psm = a.complex_obj ? d_psmice.p : nullptr;  // complex: per-pair sums in the pick
    a.snt = d_snt.p;
    a.sn_pos = d_snpos.p;
    a.mem_off = d_memoff.p;
    a.mem_list = d_memlist.p;
    a.mem_tmp = d_memtmp.p;
    a.rank = comm ? rank : 0;
    a.world = comm ? world : 1;
    a.xch = comm ? 1 : 0;
    a.dcomm = dcomm;
    a.win = win;
    a.rec_bytes = rec_bytes;
    a.xemul = (comm && world == 1) ? xemul : 1;
    a.has_target = cfg.target_reduction ? 1 : 0;
    a.target = cfg.target_reduction ? *cfg.target_reduction : 0.0;
    a.br_from = d_brf.p;
    a.br_to = d_brt.p;
    a.mask = d_mask.p;
    a.prow_off = d_prow_off.p;
    a.sup = d_sup.p;
    a.sn = d_sn.p;
    a.tab_of_node = d_tabnode.p;
    a.tab = d_tab.p;
    a.tplain = d_tplain.p;
    a.cs = d_cs.p;
    a.cr = d_cr.p;
    a.cand = d_cand.p;
    a.cidx = d_cidx.p;
    a.pcand = d_pcand.p;
    a.pmaxerr = d_pmaxerr.p;
    a.iagg = d_iagg.p;
    a.bv = d_bv.p;
    a.iaggp = d_iaggp.p;
    a.tr_sr = d_trsr.p;
    a.tr_c = d_trc.p;
    a.tr_smice = d_trsmice.p;
    a.tr_me = d_trme.p;
    a.tr_t = d_trt.p;
    return a;
  }

  bool pdl = std::getenv("KRONRED_NO_PDL") == nullptr;
  bool pdl_score = std::getenv("KRONRED_PDL_SCORE") != nullptr;
  template <class... P, class... A>
  void launch_dep(bool on, void (*k)(P...), dim3 g, dim3 b, size_t smem, cudaStream_t st, A... args) {
    cudaLaunchConfig_t c{};
    c.gridDim = g;
    c.blockDim = b;
    c.dynamicSmemBytes = smem;
    c.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    c.attrs = at;
    c.numAttrs = on ? 1 : 0;
    CK(cudaLaunchKernelEx(&c, k, args...));
  }

  // After begin(): runs every iteration on the device (one graph launch with
  // a conditional WHILE node) and returns the committed trace.
  // live: a row callback (s, r, candidates, smice, max_err[L], wall_ms) invoked
  // on the calling thread while the graph runs, in commit order; the returned
  // arrays are then left empty
  using LiveFn = std::function<void(int, int, int, double, const double*, double)>;
  char* h_live = nullptr;  // mapped host memory: count + rows
  size_t h_live_cap = 0;
  void run_device_loop(std::vector<int>& tr_s, std::vector<int>& tr_r, std::vector<int>& tr_c,
                       std::vector<double>& tr_smice, std::vector<double>& tr_me, std::vector<double>& tr_ms,
                       const LiveFn* live = nullptr) {
    const int nb = int(prob.net.branches.size());
    if (!stream2) {
      CK(cudaStreamCreateWithFlags(&stream2, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
      CK(cudaFuncSetAttribute(enum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(enum_smem())));
    }
    d_loopst.alloc(1);
    d_snpos.alloc(size_t(n));
    d_memtmp.alloc(size_t(n));
    d_sup.alloc(size_t(n));
    d_sn.alloc(size_t(n));
    d_tabnode.alloc(size_t(n));
    d_brf.alloc(size_t(nb) + 1);
    d_brt.alloc(size_t(nb) + 1);
    d_trsr.alloc(size_t(2 * n));
    d_trc.alloc(size_t(n));
    d_trsmice.alloc(size_t(n));
    d_trme.alloc(size_t(n) * L);
    d_trt.alloc(size_t(n) + 1);
    d_cand.alloc(size_t(2 * nb) + 1);
    d_cidx.alloc(size_t(2 * nb) + 1);
    d_pcand.alloc(size_t(2 * nb) + 1);
    d_pmaxerr.alloc((size_t(2 * nb) + 1) * L);
    {
      std::vector<int> ident(static_cast<size_t>(n)), bf(static_cast<size_t>(nb)), bt(static_cast<size_t>(nb));
      std::iota(ident.begin(), ident.end(), 0);
      for (int b = 0; b < nb; ++b) {
        bf[size_t(b)] = prob.net.branches[size_t(b)].from;
        bt[size_t(b)] = prob.net.branches[size_t(b)].to;
      }
      CK(cudaMemcpyAsync(d_sup.p, ident.data(), sizeof(int) * size_t(n), cudaMemcpyHostToDevice, stream));
      if (cfg.objective == Objective::complex_error) {  // every node its own cluster
        std::vector<int> off(static_cast<size_t>(n) + 1);
        std::iota(off.begin(), off.end(), 0);
        CK(cudaMemcpyAsync(d_memlist.p, ident.data(), sizeof(int) * size_t(n), cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(d_memoff.p, off.data(), sizeof(int) * (size_t(n) + 1), cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));  // pageable sources
      }
      CK(cudaMemcpyAsync(d_sn.p, ident.data(), sizeof(int) * size_t(n), cudaMemcpyHostToDevice, stream));
      if (nb) {
        CK(cudaMemcpyAsync(d_brf.p, bf.data(), sizeof(int) * size_t(nb), cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(d_brt.p, bt.data(), sizeof(int) * size_t(nb), cudaMemcpyHostToDevice, stream));
      }
      LoopState st0{};
      st0.done = target_reached() ? 1 : 0;
      st0.ns = n;
      // pageable sources: cudaMemcpyAsync stages them before returning
      CK(cudaMemcpyAsync(d_loopst.p, &st0, sizeof st0, cudaMemcpyHostToDevice, stream));
    }
    LoopArgs la = loop_args();
    // live rows: [count (64 B)] [src cap*3 int] [smice cap] [me cap*L] [t cap]
    const size_t live_bytes = 64 + size_t(n) * (3 * sizeof(int) + sizeof(double) * (1 + size_t(L)) + 8) + 64;
    if (live) {
      if (!h_live || h_live_cap < live_bytes) {
        if (h_live) CK(cudaFreeHost(h_live));
        h_live = nullptr;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&h_live), live_bytes, cudaHostAllocMapped));
        h_live_cap = live_bytes;
      }
      std::memset(h_live, 0, 64);
      char* dp = nullptr;
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), h_live, 0));
      size_t o = 64;
      la.live_count = reinterpret_cast<volatile int*>(dp);
      la.live_src = reinterpret_cast<int*>(dp + o);
      o += size_t(n) * 3 * sizeof(int);
      o = (o + 7) & ~size_t(7);
      la.live_smice = reinterpret_cast<double*>(dp + o);
      o += size_t(n) * sizeof(double);
      la.live_me = reinterpret_cast<double*>(dp + o);
      o += size_t(n) * L * sizeof(double);
      la.live_t = reinterpret_cast<unsigned long long*>(dp + o);
    }
    if (loop_trace) {
      d_tdbg.alloc(size_t(n + 1) * kTdbg);
      CK(cudaMemsetAsync(d_tdbg.p, 0, sizeof(unsigned long long) * size_t(n + 1) * kTdbg, stream));
      la.tdbg = d_tdbg.p;
    }
    BaseArgs bb = full.bprog;
    bb.L = L;
    bb.W = full.bW;
    bb.cfac = full.cfac.p;
    bb.meta = full.bmeta.p;
    bb.iaggp = d_iaggp.p;
    bb.kept_val = d_slackv.p;
    bb.bv = d_bv.p;
    bb.dbg = nullptr;
    bb.st = d_loopst.p;
    bb.tdbg = la.tdbg;
    bb.tfwd = bb.walk >= 0 ? d_tfwd.p : nullptr;
    bb.inc = (bb.walk >= 0 && !force_full_refresh) ? 1 : 0;
    // first enumeration (also stamps the loop start)
    enum_kernel<<<1, kLoopThreads, enum_smem(), stream>>>(la);
    launched();
    CK(cudaGetLastError());
    const void* bufs[kLoopKeyBufs] = {d_bv.p,   d_iagg.p, d_pmaxerr.p, d_tfwd.p,   d_cs.p,   d_cr.p,
                                      d_cand.p, d_cidx.p, d_pcand.p,   d_iaggp.p,  d_tab.p,  d_tplain.p,
                                      d_Z.p,    d_psmice.p, d_grpdone.p, d_loopst.p, d_trme.p, d_sup.p};
    const bool key_ok = loop_exec && loop_key_ebar == cfg.e_bar && loop_key_has == la.has_target &&
                        loop_key_target == la.target && loop_key_trace == loop_trace && loop_key_L == L &&
                        loop_key_live == (la.live_count != nullptr) && loop_key_comm == comm &&
                        loop_key_cplx == la.complex_obj &&
                        std::equal(bufs, bufs + kLoopKeyBufs, loop_key_bufs);
    if (!key_ok) {
      if (loop_exec) CK(cudaGraphExecDestroy(loop_exec));
      if (loop_graph) CK(cudaGraphDestroy(loop_graph));
      loop_exec = nullptr;
      loop_graph = nullptr;
      cudaGraph_t graph;
      CK(cudaGraphCreate(&graph, 0));
      cudaGraphConditionalHandle h;
      CK(cudaGraphConditionalHandleCreate(&h, graph, 1u, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp{};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t cnode;
      CK(cudaGraphAddNode(&cnode, graph, nullptr, 0, &cp));
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      LoopArgs lb = la;
      lb.use_cond = 1;
      lb.cond = h;
      CK(cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      // kLoopUnroll iterations per body execution: the conditional relaunch
      // costs a few microseconds, and iterations after the last one are
      // early-exit no-ops (every kernel checks st->done)
      // score3 grid: persistent over work items, sized for the largest candidate set
      S3Args q = s3_args();
      q.st = d_loopst.p;
      q.tdbg = la.tdbg;
      int occ = 0;
      const size_t sm3 = S3Layout{s3_ls(), s3_slots()}.smem_bytes();
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, score3_kernel<0>, s3_threads(), sm3));
      int sms = 0;
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
      const int items_max = 4 * ((2 * nb + 4) / 5 + 3) * s3_nsl();  // up to 4 lanes per pair
      const int grid3 = std::max(1, std::min(items_max, std::max(1, occ) * sms));
      size_t sm3s[3] = {sm3, sm3, sm3};
      int grid3s[3] = {grid3, grid3, grid3};
      for (int i = 1; i < 3 && !std::getenv("KRONRED_S3_FULL_SMEM"); ++i) {
        sm3s[i] = S3Layout{s3_ls(), s3_slots(), i == 1 ? 2 : 4, S3_NS_SPLIT}.smem_bytes();
        int oc = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, score3_kernel<0>, s3_threads(), sm3s[i]));
        grid3s[i] = std::max(1, std::min(items_max, std::max(1, oc) * sms));
      }
      const bool cplx = cfg.objective == Objective::complex_error;
      const bool s1 = s1_ok() && !cplx;  // (every created handle must drive a node)
      // one switch handle per unrolled copy (a handle drives one conditional
      // node); the enumeration of copy u sets copy u + 1's
      cudaGraphConditionalHandle hsw[kLoopUnroll] = {};
      if (!cplx) {
        // first iteration's split: the candidate count of iteration 1 is a
        // property of the network (the graph is keyed on it)
        std::vector<int> c0s, c0r;
        hs.enumerate(c0s, c0r);
        const int S0 = s3_lanes((long long)c0s.size() * L, s3_fill(), s3_force, s3_fill4_16());
        for (int u = 0; u < kLoopUnroll; ++u)
          CK(cudaGraphConditionalHandleCreate(&hsw[u], body, unsigned(u == 0 ? s1_switch_index(S0) : 0),
                                              cudaGraphCondAssignDefault));
        lb.use_scond = 1;
        q.skip_nl1 = s1 ? 1 : 0;
        if (!stream3) {
          CK(cudaStreamCreateWithFlags(&stream3, cudaStreamNonBlocking));
          CK(cudaEventCreateWithFlags(&ev_fork3, cudaEventDisableTiming));
          CK(cudaEventCreateWithFlags(&ev_join3, cudaEventDisableTiming));
        }
      }
      ScoreArgs qc{};
      int gridc = 0, threadsc = 0;
      size_t smemc = 0;
      if (cplx) {
        qc = members_args(int(2 * nb + 1));
        if (const char* e = std::getenv("KRONRED_CPLX_K")) qc.K = std::max(1, std::atoi(e));  // tuning aid
        qc.st = d_loopst.p;
        qc.ldc = s3_ldc();
        qc.cidx = d_cidx.p;
        const int P = qc.G * L;
        threadsc = P * qc.S;
        smemc = size_t(std::max(qc.K, qc.S)) * size_t(P) * sizeof(double);
        int occc = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occc, score_kernel<true>, threadsc, smemc));
        gridc = std::max(1, std::min((2 * nb + qc.G) / qc.G, std::max(1, occc) * sms));
      }
      for (int u = 0; u < kLoopUnroll; ++u) {
      if (cplx) {
        score_kernel<true><<<gridc, threadsc, smemc, stream>>>(qc);
      } else if (s1) {
        // |phi(r)| >= 2 candidates (score3) next to the |phi(r)| = 1 ones
        // (score1<S>, S picked by the enumeration through a switch node)
        CK(cudaEventRecord(ev_fork3, stream));
        CK(cudaStreamWaitEvent(stream3, ev_fork3, 0));
        {
          // the multi-phase items are few and latency-bound (each walks every
          // row): highest priority, so their CTAs are resident before the
          // wide score1 grid fills the SMs
          cudaLaunchConfig_t lc{};
          lc.gridDim = dim3(grid3);
          lc.blockDim = dim3(s3_threads());
          lc.dynamicSmemBytes = sm3;
          lc.stream = stream3;
          cudaLaunchAttribute at[1];
          int lo = 0, hi = 0;
          CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
          at[0].id = cudaLaunchAttributePriority;
          at[0].val.priority = std::getenv("KRONRED_NO_PRIO") ? lo : hi;
          lc.attrs = at;
          lc.numAttrs = 1;
          CK(cudaLaunchKernelEx(&lc, score3_kernel<0>, q));
        }
        lb.scond = hsw[(u + 1) % kLoopUnroll];  // set by this copy's enumeration
        add_switch(stream, hsw[u], [&](int i, cudaStream_t cs) {
          const int Si = i == 0 ? 1 : (i == 1 ? 2 : 4);
          launch_s1(Si, q, s1_grid(Si, items_max), cs);
        });
        CK(cudaEventRecord(ev_join3, stream3));
        CK(cudaStreamWaitEvent(stream, ev_join3, 0));
      } else {
        // every candidate in score3: the split picks the compiled S = 1 kernel
        // or the run-time split one
        lb.scond = hsw[(u + 1) % kLoopUnroll];
        add_switch(stream, hsw[u], [&](int i, cudaStream_t cs) {
          if (i == 0)
            score3_kernel<1><<<grid3, s3_threads(), sm3, cs>>>(q);
          else  // S lanes per pair stage Z for G / S slots: a smaller CTA, a wider persistent grid
            score3_kernel<0><<<grid3s[i], s3_threads(), sm3s[i], cs>>>(q);
          launched();
          CK(cudaGetLastError());
        });
      }
      // pick and refresh follow their stream predecessor by programmatic
      // dependent launch (launch overlapped with the predecessor's tail; each
      // waits on griddepcontrol before reading its results)
      launch_dep(pdl && !s1 && !cplx, pick_commit_kernel, dim3(1), dim3(kLoopThreads), 0, stream, lb);
      CK(cudaEventRecord(ev_fork, stream));
      CK(cudaStreamWaitEvent(stream2, ev_fork, 0));
      enum_kernel<<<1, kLoopThreads, enum_smem(), stream2>>>(lb);
      const dim3 rg((L + bb.W - 1) / bb.W), rb(32 * bb.W * bb.WB);
      if (full.bsm)
        launch_dep(pdl, base_refresh_kernel<true>, rg, rb, size_t(full.bsmem), stream, bb);
      else
        launch_dep(pdl, base_refresh_kernel<false>, rg, rb, size_t(full.bsmem), stream, bb);
      CK(cudaEventRecord(ev_join, stream2));
      CK(cudaStreamWaitEvent(stream, ev_join, 0));
      }
      CK(cudaStreamEndCapture(stream, &body));
      CK(cudaGraphInstantiate(&loop_exec, graph, 0));
      loop_graph = graph;
      loop_key_ebar = cfg.e_bar;
      loop_key_has = la.has_target;
      loop_key_target = la.target;
      loop_key_trace = loop_trace;
      loop_key_L = L;
      loop_key_live = la.live_count != nullptr;
      loop_key_comm = comm;
      loop_key_cplx = la.complex_obj;
      std::copy(bufs, bufs + kLoopKeyBufs, loop_key_bufs);
    }
    // the whole loop: one graph launch (a loop that is already done runs one
    // body of early-exit kernels); results come back with one sync
    CK(cudaGraphLaunch(loop_exec, stream));
    if (live) {
      // deliver rows as the device publishes them (mapped memory, polled)
      const volatile int* cnt = reinterpret_cast<const volatile int*>(h_live);
      const int* src = reinterpret_cast<const int*>(h_live + 64);
      size_t o = 64 + size_t(n) * 3 * sizeof(int);
      o = (o + 7) & ~size_t(7);
      const double* smv = reinterpret_cast<const double*>(h_live + o);
      const double* mev = reinterpret_cast<const double*>(h_live + o + size_t(n) * sizeof(double));
      const unsigned long long* tv =
          reinterpret_cast<const unsigned long long*>(h_live + o + size_t(n) * sizeof(double) * (1 + size_t(L)));
      int done = 0;
      unsigned long long tprev = 0;  // iteration 1: from the loop start the first enumeration stamps
      for (int k = 0; k < 1000 && tprev == 0; ++k) {
        tprev = *reinterpret_cast<const volatile unsigned long long*>(h_live + 8);
        if (tprev == 0) std::this_thread::sleep_for(std::chrono::microseconds(5));
      }
      for (;;) {
        const cudaError_t q = cudaStreamQuery(stream);
        if (q != cudaSuccess && q != cudaErrorNotReady) CK(q);
        const int c = *cnt;
        std::atomic_thread_fence(std::memory_order_acquire);
        for (; done < c; ++done) {
          const double wall = tprev ? double(tv[done] - tprev) * 1e-6 : 0.0;
          tprev = tv[done];
          (*live)(src[3 * done], src[3 * done + 1], src[3 * done + 2], smv[done], mev + size_t(done) * L, wall);
        }
        if (q == cudaSuccess && *cnt == done) break;
        if (q != cudaSuccess) std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
    }
    if (!h_loopst) CK(cudaMallocHost(&h_loopst, sizeof(LoopState)));
    if (!h_trace || h_trace_cap < trace_bytes()) {  // a reload may bring more scenarios
      if (h_trace) CK(cudaFreeHost(h_trace));
      h_trace = nullptr;
      CK(cudaMallocHost(&h_trace, trace_bytes()));
      h_trace_cap = trace_bytes();
    }
    CK(cudaMemcpyAsync(h_loopst, d_loopst.p, sizeof(LoopState), cudaMemcpyDeviceToHost, stream));
    {
      char* p = h_trace;
      CK(cudaMemcpyAsync(p, d_trsr.p, sizeof(int) * 2 * size_t(n), cudaMemcpyDeviceToHost, stream));
      p += sizeof(int) * 2 * size_t(n);
      CK(cudaMemcpyAsync(p, d_trc.p, sizeof(int) * size_t(n), cudaMemcpyDeviceToHost, stream));
      p += sizeof(int) * size_t(n);
      CK(cudaMemcpyAsync(p, d_trsmice.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, stream));
      p += sizeof(double) * size_t(n);
      CK(cudaMemcpyAsync(p, d_trme.p, sizeof(double) * size_t(n) * L, cudaMemcpyDeviceToHost, stream));
      p += sizeof(double) * size_t(n) * L;
      CK(cudaMemcpyAsync(p, d_trt.p, sizeof(unsigned long long) * (size_t(n) + 1), cudaMemcpyDeviceToHost, stream));
    }
    CK(cudaStreamSynchronize(stream));
    check_deferred_fail();
    const LoopState st = *h_loopst;
    // kernels per loop-body iteration: scorer(s), pick, enumeration, refresh
    launches += (s1_ok() && cfg.objective == Objective::magnitude ? 5LL : 4LL) * ((st.iter + kLoopUnroll) / kLoopUnroll * kLoopUnroll);
    const int it = st.iter;
    if (loop_trace && it > 2) {
      std::vector<unsigned long long> T(size_t(n + 1) * kTdbg);
      CK(cudaMemcpy(T.data(), d_tdbg.p, sizeof(unsigned long long) * T.size(), cudaMemcpyDeviceToHost));
      if (const char* dump = std::getenv("KRONRED_LOOP_TRACE_DUMP")) {  // raw stamps [n+1][8] for tools/
        if (FILE* f = std::fopen(dump, "wb")) {
          std::fwrite(T.data(), sizeof(unsigned long long), size_t(it + 1) * kTdbg, f);
          std::fclose(f);
        }
      }
      // per iteration i: score start [i][6], pick [i][0..1], enum for i+1 [i+1][2..3], refresh [i+1][4..5]
      double a_sc = 0, a_pick = 0, a_p2e = 0, a_enum = 0, a_p2r = 0, a_r2s = 0, a_e2s = 0, a_ref = 0, a_tab = 0;
      int cnt = 0;
      for (int i = 1; i + 1 < it; ++i) {
        const unsigned long long* c = &T[size_t(i) * kTdbg];
        const unsigned long long* nx = &T[size_t(i + 1) * kTdbg];
        a_sc += double(c[0] - c[6]);
        a_pick += double(c[1] - c[0]);
        a_p2e += double(nx[2] - c[1]);
        a_enum += double(nx[3] - nx[2]);
        a_p2r += double(nx[4] - c[1]);
        a_r2s += double(nx[6] - nx[4]);
        a_e2s += double(nx[6] - nx[3]);
        a_ref += double(nx[5] - nx[4]);
        a_tab += double(nx[7] - nx[2]);
        ++cnt;
      }
      std::fprintf(stderr,
                   "loop timeline (us/iter avg over %d): score+gap %.1f | pick %.1f | pick->enum %.1f enum %.1f (table %.1f) | "
                   "pick->refresh %.1f refresh-start->next score %.1f (refresh block0 %.1f) | enum-end->next score %.1f\n",
                   cnt, a_sc / cnt / 1e3, a_pick / cnt / 1e3, a_p2e / cnt / 1e3, a_enum / cnt / 1e3, a_tab / cnt / 1e3,
                   a_p2r / cnt / 1e3,
                   a_r2s / cnt / 1e3, a_ref / cnt / 1e3, a_e2s / cnt / 1e3);
    }
    tr_s.resize(size_t(it));
    tr_r.resize(size_t(it));
    tr_c.resize(size_t(it));
    tr_smice.resize(size_t(it));
    tr_me.resize(size_t(it) * L);
    tr_ms.assign(size_t(it), 0.0);
    if (it > 0) {
      const char* p = h_trace;
      const int* sr = reinterpret_cast<const int*>(p);
      p += sizeof(int) * 2 * size_t(n);
      std::memcpy(tr_c.data(), p, sizeof(int) * size_t(it));
      p += sizeof(int) * size_t(n);
      std::memcpy(tr_smice.data(), p, sizeof(double) * size_t(it));
      p += sizeof(double) * size_t(n);
      std::memcpy(tr_me.data(), p, sizeof(double) * size_t(it) * L);
      p += sizeof(double) * size_t(n) * L;
      const unsigned long long* tt = reinterpret_cast<const unsigned long long*>(p);
      for (int i = 0; i < it; ++i) {
        tr_s[size_t(i)] = sr[2 * i];
        tr_r[size_t(i)] = sr[2 * i + 1];
        tr_ms[size_t(i)] = double(tt[i] - (i > 0 ? tt[i - 1] : tt[n])) * 1e-6;
      }
    }
  }

  size_t trace_bytes() const {
    return size_t(n) * (sizeof(int) * 3 + sizeof(double) * (1 + size_t(L))) +
           (size_t(n) + 1) * sizeof(unsigned long long);
  }
  LoopState* h_loopst = nullptr;
  char* h_trace = nullptr;
  size_t h_trace_cap = 0;

  void commit_device(int s, int r) {
    const unsigned ms = prob.mask[size_t(s)], mr = prob.mask[size_t(r)];
    commit_kernel<<<(L + 127) / 128, 128, 0, stream>>>(s, r, L, ms, mr, prow_off[size_t(s)], prow_off[size_t(r)],
                                                       d_iagg.p, d_bv.p, d_iaggp.p, nphi);
    launched();
    CK(cudaGetLastError());
    refresh_base(s, r);
  }
};

// ---------------------------------------------------------------------------

Engine::Engine(const Problem& prob, int device) : impl_(std::make_unique<Impl>(prob, device)) {}
Engine::~Engine() = default;

void Engine::set_profile(bool on) {
  impl_->ensure_events();
  impl_->profile = on;
  impl_->score_stats = KernelStats{};
  impl_->solve_stats = KernelStats{};
  impl_->multi_stats = KernelStats{};
}
KernelStats Engine::stats(int which) const {
  return which == 0 ? impl_->score_stats : (which == 1 ? impl_->solve_stats : impl_->multi_stats);
}
const Problem& Engine::problem() const { return impl_->prob; }
std::int64_t Engine::launches() const { return impl_->launches; }
bool Engine::last_run_device_loop() const { return impl_->last_device_loop; }

void Engine::set_comm(int rank, int world, const void* unique_id) {
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof id);
  impl_->set_comm(rank, world, id);
}

void Engine::set_exchange(int rank, int world, krg_exchange_fn fn, void* user) {
  if (world < 1 || rank < 0 || rank >= world) throw ConfigError("bad rank/world");
  impl_->rank = rank;
  impl_->world = world;
  impl_->xfn = fn;
  impl_->xuser = user;
}

const std::vector<double>& Engine::vhat() const { return impl_->h_vhat; }

void Engine::scenario_voltages(double* out) {
  std::memcpy(out, impl_->h_vhat.data(), impl_->h_vhat.size() * sizeof(double));
}

void Engine::solve(const double* inj, int nrhs, double* out) {
  Impl& I = *impl_;
  DBuf<double2> rhs, res;
  rhs.alloc(size_t(nrhs) * 3 * I.n);
  res.alloc(size_t(nrhs) * 3 * I.n);
  CK(cudaMemcpyAsync(rhs.p, inj, size_t(nrhs) * 3 * I.n * sizeof(double2), cudaMemcpyHostToDevice, I.stream));
  I.solve_full(I.full, I.d_slackv.p, rhs.p, nrhs, res.p);
  CK(cudaMemcpyAsync(out, res.p, size_t(nrhs) * 3 * I.n * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
}

void Engine::loop_begin(const ReductionConfig& cfg) {
  impl_->begin(cfg);
  CK(cudaStreamSynchronize(impl_->stream));
  impl_->check_deferred_fail();
}

void Engine::debug_base_refresh(int reps, double* ms, long long* clocks) {
  Impl& I = *impl_;
  DBuf<long long> dbg;
  dbg.alloc(4);
  CK(cudaMemset(dbg.p, 0, 4 * sizeof(long long)));
  I.ensure_events();
  // reps < 0: time the incremental refresh after the first candidate's
  // commit pattern (the walk from its s and r; values are not meaningful)
  const bool inc = reps < 0;
  if (inc) reps = -reps;
  const int s = inc && !I.cs.empty() ? I.cs[0] : -1, r = inc && !I.cr.empty() ? I.cr[0] : -1;
  I.refresh_base();
  CK(cudaEventRecord(I.ev_a, I.stream));
  for (int i = 0; i < reps; ++i) I.refresh_base(s, r);
  *ms = I.event_ms() / reps;
  I.dbg_clock = dbg.p;
  I.refresh_base(s, r);
  CK(cudaStreamSynchronize(I.stream));
  I.dbg_clock = nullptr;
  CK(cudaMemcpy(clocks, dbg.p, 4 * sizeof(long long), cudaMemcpyDeviceToHost));
}

void Engine::reload(const Problem& p) {
  // same network structure (node masks, branch endpoints, block pattern):
  // new admittance values go straight into the resident buffers; the
  // elimination schedule, loop graph and all allocations are kept
  Impl& I = *impl_;
  if (p.y.n != I.prob.y.n || p.mask != I.prob.mask || p.slack != I.prob.slack || p.y.row != I.prob.y.row ||
      p.y.col != I.prob.y.col || p.net.branches.size() != I.prob.net.branches.size())
    throw ValidationError("reload: the network structure differs from the context's");
  for (size_t b = 0; b < p.net.branches.size(); ++b)
    if (p.net.branches[b].from != I.prob.net.branches[b].from || p.net.branches[b].to != I.prob.net.branches[b].to)
      throw ValidationError("reload: the branch list differs from the context's");
  const std::vector<std::string> ids = I.prob.scenario_ids;
  I.prob = p;
  I.prob.scenario_ids = ids;
  I.prob.L = I.L;
  I.h2d_staged(I.d_yin.p, p.y.val.data(), p.y.val.size() * sizeof(double));
  double sv[6];
  for (int q = 0; q < 3; ++q) {
    sv[2 * q] = p.net.nodes[size_t(p.slack)].slack_voltage[q].real();
    sv[2 * q + 1] = p.net.nodes[size_t(p.slack)].slack_voltage[q].imag();
  }
  CK(cudaMemcpyAsync(I.d_slackv.p, sv, sizeof sv, cudaMemcpyHostToDevice, I.stream));
  I.pivot_floor = 1e-12 * std::max(p.y.max_abs(), 1.0);
  I.factorize(I.full, I.d_yin.p, I.pivot_floor);
}

void Engine::set_scenarios(const std::vector<std::string>& ids, const std::vector<double>& inj,
                           const std::vector<double>& volt) {
  impl_->load_scenarios(ids, inj, volt);
}

void Engine::pq_to_currents(const std::vector<std::vector<std::pair<int, cx>>>& loads, std::vector<double>& inj,
                            std::vector<double>& volt) {
  // scenario_from_pq (scenario.cpp:52-98): I = -conj(S/V) fixed point, one
  // device anchored solve per sweep, all scenarios batched; each scenario
  // stops at its own convergence like the reference's per-scenario loop.
  Impl& I = *impl_;
  const int n = I.n;
  const int L = int(loads.size());
  const size_t dim = size_t(3 * n);
  std::vector<cx> v0(dim);
  {
    DBuf<double2> out;
    out.alloc(dim);
    I.solve_full(I.full, I.d_slackv.p, nullptr, 1, out.p);
    CK(cudaMemcpyAsync(v0.data(), out.p, dim * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
    CK(cudaStreamSynchronize(I.stream));
  }
  const std::vector<cx> zeros(dim);
  std::vector<std::vector<cx>> S(static_cast<size_t>(L), zeros), V(static_cast<size_t>(L), v0), J(static_cast<size_t>(L), zeros);
  for (int l = 0; l < L; ++l)
    for (const auto& ld : loads[size_t(l)]) S[size_t(l)][size_t(ld.first)] += ld.second;
  std::vector<char> done(size_t(L), 0);
  std::vector<double> last_dv(size_t(L), 0.0);
  DBuf<double2> d_rhs, d_out;
  d_rhs.alloc(dim * size_t(std::max(L, 1)));
  d_out.alloc(dim * size_t(std::max(L, 1)));
  std::vector<cx> rhs(dim * size_t(L)), res(dim * size_t(L));
  for (int it = 0; it < 50; ++it) {
    std::vector<int> act;
    for (int l = 0; l < L; ++l)
      if (!done[size_t(l)]) act.push_back(l);
    if (act.empty()) break;
    for (size_t a = 0; a < act.size(); ++a) {
      const int l = act[a];
      for (size_t k = 0; k < dim; ++k) {
        const cx sk = S[size_t(l)][k];
        if (sk == cx{}) continue;
        if (std::abs(V[size_t(l)][k]) < 1e-6)
          throw SolverError("scenario '" + I.prob.scenario_ids[size_t(l)] + "': voltage collapse during PQ conversion");
        J[size_t(l)][k] = -std::conj(sk / V[size_t(l)][k]);
      }
      std::copy(J[size_t(l)].begin(), J[size_t(l)].end(), rhs.begin() + long(a * dim));
    }
    CK(cudaMemcpyAsync(d_rhs.p, rhs.data(), act.size() * dim * sizeof(double2), cudaMemcpyHostToDevice, I.stream));
    I.solve_full(I.full, I.d_slackv.p, d_rhs.p, int(act.size()), d_out.p);
    CK(cudaMemcpyAsync(res.data(), d_out.p, act.size() * dim * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
    CK(cudaStreamSynchronize(I.stream));
    for (size_t a = 0; a < act.size(); ++a) {
      const int l = act[a];
      double dv = 0;
      for (size_t k = 0; k < dim; ++k) dv = std::max(dv, std::abs(res[a * dim + k] - V[size_t(l)][k]));
      std::copy(res.begin() + long(a * dim), res.begin() + long((a + 1) * dim), V[size_t(l)].begin());
      last_dv[size_t(l)] = dv;
      if (dv < 1e-9) done[size_t(l)] = 1;
    }
  }
  for (int l = 0; l < L; ++l)
    if (!done[size_t(l)])
      throw SolverError("scenario '" + I.prob.scenario_ids[size_t(l)] +
                        "': PQ fixed point did not converge in 50 iterations");
  inj.assign(dim * 2 * size_t(L), 0.0);
  volt.assign(dim * 2 * size_t(L), 0.0);
  for (int l = 0; l < L; ++l)
    for (size_t k = 0; k < dim; ++k) {
      inj[(size_t(l) * dim + k) * 2] = J[size_t(l)][k].real();
      inj[(size_t(l) * dim + k) * 2 + 1] = J[size_t(l)][k].imag();
      volt[(size_t(l) * dim + k) * 2] = V[size_t(l)][k].real();
      volt[(size_t(l) * dim + k) * 2 + 1] = V[size_t(l)][k].imag();
    }
}

std::int64_t Engine::loop_candidates(std::vector<int>& cs, std::vector<int>& cr) {
  Impl& I = *impl_;
  if (!I.loop_active) throw Error("loop not started");
  I.hs.enumerate(I.cs, I.cr);
  cs = I.cs;
  cr = I.cr;
  return std::int64_t(I.cs.size());
}

void Engine::loop_score_all(double* smice, std::uint8_t* feasible, double* max_err) {
  Impl& I = *impl_;
  const long long C = (long long)I.cs.size();
  I.upload_iteration(0, C);
  I.launch_score(C);
  // score3 writes scenario-major [L][ldc]; the complex scorer candidate-major [C][L]
  const bool tr = !I.cfg.use_delta || I.cfg.objective == Objective::magnitude;
  const size_t ldc = size_t(I.s3_ldc());
  const size_t npair = tr ? ldc * I.L : size_t(C) * I.L;
  std::vector<double> ps(npair), pm(npair);
  if (C > 0) {
    CK(cudaMemcpyAsync(ps.data(), I.d_psmice.p, ps.size() * sizeof(double), cudaMemcpyDeviceToHost, I.stream));
    CK(cudaMemcpyAsync(pm.data(), I.d_pmaxerr.p, pm.size() * sizeof(double), cudaMemcpyDeviceToHost, I.stream));
  }
  CK(cudaStreamSynchronize(I.stream));
  for (long long c = 0; c < C; ++c) {
    bool feas = true;
    double sum = 0;
    for (int l = 0; l < I.L; ++l) {
      const size_t o = tr ? size_t(l) * ldc + size_t(c) : size_t(c) * I.L + l;
      feas = feas && !(pm[o] > I.cfg.e_bar);
      sum += ps[o];
      if (max_err) max_err[size_t(c) * I.L + l] = pm[o];
    }
    feasible[c] = feas ? 1 : 0;
    smice[c] = feas ? sum : std::numeric_limits<double>::infinity();
  }
}

void Engine::loop_best(krg_best* out, double* max_err) {
  Impl& I = *impl_;
  int64_t c0 = 0, c1 = (int64_t)I.cs.size();
  if (I.world > 1) krg_shard_range(c1, I.rank, I.world, &c0, &c1);
  I.score_best(c0, c1);
  I.exchange_best();
  const long long idx = I.best_index();
  out->index = idx;
  out->smice = idx < 0 ? std::numeric_limits<double>::infinity() : I.h_best[0];
  out->s = idx < 0 ? -1 : I.cs[size_t(idx)];
  out->r = idx < 0 ? -1 : I.cr[size_t(idx)];
  if (max_err) std::memcpy(max_err, I.h_best + 2, sizeof(double) * size_t(I.L));
}

void Engine::loop_commit(int s, int r) {
  Impl& I = *impl_;
  I.hs.commit(s, r);
  I.commit_device(s, r);
  CK(cudaStreamSynchronize(I.stream));
}

void Engine::loop_base(double* out) {
  Impl& I = *impl_;
  std::vector<double2> bv(size_t(I.nphi) * I.L * 2);
  CK(cudaMemcpyAsync(bv.data(), I.d_bv.p, bv.size() * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
  std::memset(out, 0, sizeof(double) * size_t(I.L) * 6 * I.n);
  for (int r = 0; r < I.nphi; ++r)
    for (int l = 0; l < I.L; ++l) {
      const size_t o = (size_t(l) * 3 * I.n + size_t(I.prow_node[size_t(r)]) * 3 + I.prow_phase[size_t(r)]) * 2;
      out[o] = bv[bv_base(size_t(r), I.L, l)].x;
      out[o + 1] = bv[bv_base(size_t(r), I.L, l)].y;
    }
}

void Engine::zcols(double* out, std::int64_t cap) {
  Impl& I = *impl_;
  const size_t need = size_t(I.nphi) * I.nphi * 2;
  if (size_t(cap) < need) throw ValidationError("zcols: buffer too small");
  if (!I.d_Z.p) I.build_z();
  CK(cudaMemcpyAsync(out, I.d_Z.p, need * sizeof(double), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
}

void Engine::run(const ReductionConfig& cfg, const Observer& obs, ResultData& out) {
  Impl& I = *impl_;
  const auto tw0 = std::chrono::steady_clock::now();
  out = ResultData{};
  out.L = I.L;
  I.ensure_events();
  CK(cudaEventRecord(I.ev_run0, I.stream));
  I.begin(cfg);
  int iteration = 0;
  I.last_device_loop = I.device_loop_ok(cfg);
  if (!I.device_loop_ok(cfg)) {  // host-driven loop: surface a singular factorization first
    CK(cudaStreamSynchronize(I.stream));
    I.check_deferred_fail();
  }
  if (I.device_loop_ok(cfg)) {
    // whole loop on the device; the host state machine replays the commits
    // afterwards to rebuild clusters and call the observer in order
    std::vector<int> ts, tr, tc;
    std::vector<double> tsm, tme, tms;
    const char* om = std::getenv("KRONRED_OBSERVER");
    const bool live = obs && !(om && std::string(om) == "replay");
    Impl::LiveFn deliver = [&](int s, int r, int c, double smice, const double* me, double wall) {
      // the observer sees the state after this commit, on the calling thread,
      // while later iterations run on the device (reduce.cpp:406-423)
      I.hs.commit(s, r);
      TraceRow row;
      row.iteration = ++iteration;
      row.s = s;
      row.r = r;
      row.smice = smice;
      row.max_err.assign(me, me + I.L);
      row.supernode_count = int(I.hs.supernodes.size());
      row.candidate_count = c;
      row.wall_ms = wall;
      out.total_candidates += c;
      obs(I.hs, row);
      out.trace.push_back(std::move(row));
    };
    I.run_device_loop(ts, tr, tc, tsm, tme, tms, live ? &deliver : nullptr);
    if (live) ts.clear();
    for (size_t i = 0; i < ts.size(); ++i) {
      I.hs.commit(ts[i], tr[i]);
      TraceRow row;
      row.iteration = ++iteration;
      row.s = ts[i];
      row.r = tr[i];
      row.smice = tsm[i];
      row.max_err.assign(tme.begin() + long(i * size_t(I.L)), tme.begin() + long((i + 1) * size_t(I.L)));
      row.supernode_count = int(I.hs.supernodes.size());
      row.candidate_count = tc[i];
      row.wall_ms = tms[i];
      out.total_candidates += tc[i];
      if (obs) obs(I.hs, row);
      out.trace.push_back(std::move(row));
    }
  }
  while (!I.device_loop_ok(cfg) && !I.target_reached()) {
    const auto t0 = std::chrono::steady_clock::now();
    I.hs.enumerate(I.cs, I.cr);
    const long long C = (long long)I.cs.size();
    if (C == 0) break;
    int64_t c0 = 0, c1 = C;
    if (I.world > 1) krg_shard_range(C, I.rank, I.world, &c0, &c1);
    I.score_best(c0, c1);
    I.exchange_best();
    const long long best = I.best_index();
    if (best < 0) break;
    const int s = I.cs[size_t(best)], r = I.cr[size_t(best)];
    I.commit_device(s, r);
    I.hs.commit(s, r);
    TraceRow row;
    row.iteration = ++iteration;
    row.s = s;
    row.r = r;
    row.smice = I.h_best[0];
    row.max_err.assign(I.h_best + 2, I.h_best + 2 + I.L);
    row.supernode_count = int(I.hs.supernodes.size());
    row.candidate_count = int(C);
    row.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    out.total_candidates += C;
    if (obs) obs(I.hs, row);
    out.trace.push_back(std::move(row));
  }
  CK(cudaStreamSynchronize(I.stream));
  I.loop_active = false;
  // final Kron reduction over the surviving super-nodes (reduce.cpp:426-450)
  Partition part;
  part.keep = I.hs.supernodes;
  for (int i = 0; i < I.n; ++i)
    if (I.hs.sup[size_t(i)] != i) part.reduce.push_back(i);
  check_partition(part, I.n, I.prob.slack);
  ReducedModel& model = out.model;
  kron(part.reduce, model);
  for (int i : I.hs.supernodes) {
    std::vector<int> mem = I.hs.members[size_t(i)];
    std::sort(mem.begin(), mem.end());
    model.clusters[i] = std::move(mem);
  }
  model.e_bar = cfg.e_bar;
  model.objective = cfg.objective;
  model.scenario_ids = I.prob.scenario_ids;
  model.final_max_err = model_errors(model);
  out.state = I.hs;
  CK(cudaEventRecord(I.ev_run1, I.stream));
  CK(cudaEventSynchronize(I.ev_run1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, I.ev_run0, I.ev_run1));
  out.device_ms = ms;
  if (std::getenv("KRONRED_RELOAD_TRACE"))
    std::fprintf(stderr, "run: host wall %.3f ms, device %.3f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw0).count(), double(ms));
}

void Engine::kron(const std::vector<int>& reduce, ReducedModel& model) {
  Impl& I = *impl_;
  DevElim& e = I.kron_e;
  I.upload_elim(e, I.prob.y, I.prob.mask, reduce, /*with_solve=*/false);
  I.factorize(e, I.d_yin.p, 1e-12 * std::max(I.prob.y.max_abs(), 1.0));
  const ElimSchedule& h = e.h;
  std::vector<double2> blocks(size_t(h.nblocks) * 9);
  CK(cudaMemcpyAsync(blocks.data(), e.blocks.p, blocks.size() * sizeof(double2), cudaMemcpyDeviceToHost,
                     I.stream));
  CK(cudaStreamSynchronize(I.stream));
  std::vector<int> pos(size_t(I.n), -1);
  for (size_t p = 0; p < h.kept.size(); ++p) pos[size_t(h.kept[p])] = int(p);
  model.kept_ids = h.kept;
  model.kept_phases.clear();
  for (int id : h.kept) model.kept_phases.push_back(PhaseMask{I.prob.mask[size_t(id)]});
  model.y_kron = BlockMatrix(int(h.kept.size()));
  for (size_t q = 0; q < h.rem_i.size(); ++q) {
    Mat3c m;
    const int b = h.rem_blk[q];
    for (int k = 0; k < 9; ++k) {
      const double2 v = b >= 0 ? blocks[size_t(b) * 9 + k] : make_double2(0.0, 0.0);
      m.m[size_t(k)] = cx{v.x, v.y};
    }
    if (m.is_zero()) continue;
    model.y_kron.block(pos[size_t(h.rem_i[q])], pos[size_t(h.rem_j[q])]) = m;
  }
}

std::vector<double> Engine::model_errors(const ReducedModel& model) {
  // model_max_errors (reduce.cpp:490-550): anchored solve on Y_kron with
  // cluster-aggregated injections; |.| via std::abs on the host read-back.
  Impl& I = *impl_;
  const Network& net = I.prob.net;
  const int slack = I.prob.slack;
  auto pos_of = [&](int id) {
    auto it = std::lower_bound(model.kept_ids.begin(), model.kept_ids.end(), id);
    if (it == model.kept_ids.end() || *it != id)
      throw ValidationError("reduced model does not keep node " + std::to_string(id));
    return int(it - model.kept_ids.begin());
  };
  const int slack_pos = pos_of(slack);
  const int nk = int(model.kept_ids.size());
  std::vector<int> assigned(size_t(net.size()), -1);
  for (const auto& [i, mem] : model.clusters) {
    const int pi = pos_of(i);
    for (int j : mem) {
      if (j < 0 || j >= net.size()) throw ValidationError("cluster references unknown node");
      assigned[size_t(j)] = pi;
    }
  }
  for (int p = 0; p < nk; ++p) assigned[size_t(model.kept_ids[size_t(p)])] = p;
  for (int j = 0; j < net.size(); ++j)
    if (assigned[size_t(j)] < 0)
      throw ValidationError("node " + std::to_string(j) + " is not covered by any cluster");

  const FlatBlocks yk = FlatBlocks::from(model.y_kron);
  std::vector<std::uint8_t> kmask(static_cast<size_t>(nk));
  for (int p = 0; p < nk; ++p) kmask[size_t(p)] = model.kept_phases[size_t(p)].bits;
  DevElim& e = I.merr_e;
  std::vector<int> elim;
  for (int p = 0; p < nk; ++p)
    if (p != slack_pos) elim.push_back(p);
  I.upload_elim(e, yk, kmask, elim);
  DBuf<double2>& yin = I.merr_yin;
  yin.alloc(yk.row.size() * 9);
  if (!yk.row.empty())
    CK(cudaMemcpyAsync(yin.p, yk.val.data(), yk.val.size() * sizeof(double), cudaMemcpyHostToDevice, I.stream));
  I.factorize(e, yin.p, 1e-12 * std::max(yk.max_abs(), 1.0));

  const int L = I.L;
  const int n = net.size();
  std::vector<double> rhs(size_t(L) * 6 * nk, 0.0);
  for (int l = 0; l < L; ++l) {
    std::vector<cx> ik(size_t(3 * nk), cx{});
    const double* inj = I.prob.injections.data() + size_t(l) * 6 * n;
    for (const auto& [i, mem] : model.clusters) {
      const int pi = pos_of(i);
      for (int j : mem)
        for (int p = 0; p < 3; ++p) ik[size_t(3 * pi + p)] += cx{inj[(3 * j + p) * 2], inj[(3 * j + p) * 2 + 1]};
    }
    for (int t = 0; t < 3 * nk; ++t) {
      rhs[size_t(l) * 6 * nk + size_t(t) * 2] = ik[size_t(t)].real();
      rhs[size_t(l) * 6 * nk + size_t(t) * 2 + 1] = ik[size_t(t)].imag();
    }
  }
  DBuf<double2>& d_rhs = I.merr_rhs;
  DBuf<double2>& d_out = I.merr_out;
  DBuf<double2>& d_kv = I.merr_kv;
  d_rhs.alloc(size_t(L) * 3 * nk);
  d_out.alloc(size_t(L) * 3 * nk);
  CK(cudaMemcpyAsync(d_rhs.p, rhs.data(), rhs.size() * sizeof(double), cudaMemcpyHostToDevice, I.stream));
  I.solve_full(e, I.d_slackv.p, d_rhs.p, L, d_out.p);
  std::vector<double> vk(size_t(L) * 6 * nk);
  CK(cudaMemcpyAsync(vk.data(), d_out.p, vk.size() * sizeof(double), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
  std::vector<double> out;
  for (int l = 0; l < L; ++l) {
    double err = 0;
    for (int j = 0; j < n; ++j) {
      const int pj = assigned[size_t(j)];
      for (int p = 0; p < 3; ++p) {
        if (!I.prob.net.nodes[size_t(j)].phases.has(p)) continue;
        const double* a = &vk[size_t(l) * 6 * nk + size_t(3 * pj + p) * 2];
        const double* b = &I.h_vhat[size_t(l) * 6 * n + size_t(3 * j + p) * 2];
        const double e2 = std::fabs(std::abs(cx{a[0], a[1]}) - std::abs(cx{b[0], b[1]}));
        err = std::max(err, e2);
      }
    }
    out.push_back(err);
  }
  return out;
}

void Engine::radialize(ReducedModel& model, bool with_errors) {
  auto kr = [this](const std::vector<int>& reduce, ReducedModel& m) { this->kron(reduce, m); };
  std::function<std::vector<double>(const ReducedModel&)> errs = [this](const ReducedModel& m) {
    return this->model_errors(m);
  };
  model = radialize_host(model, impl_->prob.net, kr, with_errors ? &errs : nullptr);
}

extern "C" int krg_nccl_unique_id(uint8_t* out) {
  try {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw Error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(id) == KRG_NCCL_ID_BYTES, "NCCL unique id size");
    std::memcpy(out, &id, sizeof id);
    return KRG_OK;
  } catch (...) {
    return status_from_current_exception();
  }
}

// measured unfused FP64 rate (GFLOP/s, DMUL+DADD counted as 2) on `device`
extern "C" int krg_fp64_probe(int32_t device, double* gflops) {
  try {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) throw CudaError("no CUDA device");
    if (device >= 0) CK(cudaSetDevice(device));
    int sms = 0, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DBuf<double> sink;
    sink.alloc(1);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    fp64_probe_kernel<<<blocks, threads>>>(iters, 0.999999, 1e-7, sink.p);  // warm-up
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0));
      fp64_probe_kernel<<<blocks, threads>>>(iters, 0.999999, 1e-7, sink.p);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = std::max(best, 2.0 * 8.0 * iters * double(blocks) * threads / (ms * 1e-3) / 1e9);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *gflops = best;
    return KRG_OK;
  } catch (...) {
    return status_from_current_exception();
  }
}

}  // namespace kronred::b200

// debug/benchmark hook: time `reps` base refreshes (requires krg_loop_begin);
// clocks[0..3] = block-0 warp-0 timestamps (start, forward, backward, output)
extern "C" int krg_debug_base_refresh(krg_ctx* ctx, int32_t reps, double* ms, long long* clocks);

namespace kronred::b200 {

// self test: branch-free scorer sqrt vs __dsqrt_rn on n random inputs in [lo,hi)
extern "C" int krg_selftest_sqrt(int64_t n, double lo, double hi, int64_t* mismatches) {
  try {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) throw CudaError("no CUDA device");
    DBuf<unsigned long long> bad;
    bad.alloc(1);
    CK(cudaMemset(bad.p, 0, sizeof(unsigned long long)));
    selftest_sqrt_kernel<<<unsigned((n + 255) / 256), 256>>>(n, 12345ull, bad.p, lo, hi);
    CK(cudaGetLastError());
    unsigned long long h = 0;
    CK(cudaMemcpy(&h, bad.p, sizeof h, cudaMemcpyDeviceToHost));
    *mismatches = (int64_t)h;
    return KRG_OK;
  } catch (...) {
    return status_from_current_exception();
  }
}

// self test hook for the __divdc3 replica (device)
extern "C" int krg_selftest_cdiv(const double* in, int32_t N, double* out, int32_t on_device) {
  try {
    if (!on_device) {
      for (int i = 0; i < N; ++i) {
        const C2 r = dev::cdiv({in[4 * i], in[4 * i + 1]}, {in[4 * i + 2], in[4 * i + 3]});
        out[2 * i] = r.x;
        out[2 * i + 1] = r.y;
      }
      return KRG_OK;
    }
    DBuf<double> din, dout;
    din.alloc(size_t(N) * 4);
    dout.alloc(size_t(N) * 2);
    CK(cudaMemcpy(din.p, in, size_t(N) * 4 * sizeof(double), cudaMemcpyHostToDevice));
    selftest_cdiv_kernel<<<(N + 127) / 128, 128>>>(N, din.p, dout.p);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, dout.p, size_t(N) * 2 * sizeof(double), cudaMemcpyDeviceToHost));
    return KRG_OK;
  } catch (...) {
    return status_from_current_exception();
  }
}

}  // namespace kronred::b200
