// Device-resident iteration loop (magnitude objective, one GPU).
//
// The integer half of Algorithm 1 moves onto the device so that a whole
// reduction runs as one CUDA graph with a conditional WHILE node and no host
// round trip per iteration:
//
//   enum_kernel         enumerate_candidates (reduce.cpp:63-73) from the
//                       super-node map: every branch (a,b) with sup[a] != sup[b]
//                       is a super-node edge (a contracted tree has no parallel
//                       edges); both directions are filtered (r != slack,
//                       phi(r) subset of phi(s)) and sorted lexicographically
//                       (bitonic sort of (s << 16 | r) keys in shared memory).
//                       It also lays out the scorer's row table: active
//                       super-nodes ascending, rows in 4-row blocks that never
//                       split a super-node (a 4-state transducer, scanned over
//                       the block), and groups the candidates by |phi(r)|.
//   pick_commit_kernel  the argmin (reduce.cpp:397-404: first minimum SMICE among
//                       feasible candidates), the trace row, and commit
//                       (reduce.cpp:299-344): i_agg move, cluster bound merge,
//                       super-node map relabel, removal of r from the active
//                       list, target test (reduce.cpp:369-373).
//
// Every kernel of the loop body returns immediately once st->done is set;
// enum_kernel sets the graph's loop condition.
#pragma once

namespace kronred::b200 {
namespace {

struct LoopArgs {
  LoopState* st;
  int n, nb, slack, L, nphi, cap;
  int G3;              // scorer Z-column slots per CTA (candidates per CTA: s3_cpc(G3, |phi(r)|, S))
  int gk1[3];          // score1 candidates per CTA at S = 1, 2, 4 (0: score3 takes |phi(r)| = 1 too)
  int s_multi;         // score3's split for the |phi(r)| >= 2 groups when score1 runs
  long long fill;      // scorer row split: thread budget (s3_lanes)
  int fill4_16;        // S = 4 threshold in sixteenths of the budget
  int force_s;         // scorer row split forced to 1/2/4 (0: automatic)
  int inc_enum;        // 1: incremental candidate list after a commit (else full rebuild)
  int kcap;            // keys region size (power of two >= 2 nb); the previous list follows it
  int nsl;             // scenario slices per candidate group (score3), 1 otherwise
  const double* psm;   // score3 per-pair SMICE [L][ldc] (null: pcand holds per-candidate sums)
  int ldc;
  double e_bar;
  int has_target;
  double target;
  const int* br_from;
  const int* br_to;
  const std::uint8_t* mask;
  const int* prow_off;
  int* sup;            // [n] super-node of every original node
  int* sn;             // [n] active super-nodes, ascending (st->ns of them)
  int* tab_of_node;    // [n] first table row of each active super-node
  unsigned* tab;       // [4n + pad] row table
  std::uint8_t* tplain;  // [tiles of 16 rows] 1: every row a single-row super-node, no padding
  int* cs;             // [2n] candidates, lexicographic
  int* cr;
  int4* cand;          // [2n] grouped by |phi(r)|: (s, r, tab(s), tab(r))
  int* cidx;           // [2n] lexicographic index of each grouped slot
  const double* pcand; // [C] SMICE or -1 (infeasible), lexicographic index
  const double* pmaxerr;
  double2* iagg;       // [n][L][3]
  double2* bv;         // [nphi][L][2]
  double2* iaggp;      // [L][nphi]
  int* tr_sr;          // [cap][2]
  int* tr_c;           // [cap]
  double* tr_smice;    // [cap]
  double* tr_me;       // [cap][L]
  unsigned long long* tr_t;  // [cap] globaltimer at commit
  cudaGraphConditionalHandle cond;
  int use_cond;
  cudaGraphConditionalHandle scond;  // switch over the scorer's row split (score1<1|2|4>)
  int use_scond;
  unsigned long long* tdbg;  // optional timeline [iter][8]: pick start/end, enum start/end
  // live trace (observer delivery while the graph runs): rows mirrored into
  // mapped host memory, then the published row count (null: off)
  // multi-GPU (one rank per GPU): candidates of an iteration are split in
  // contiguous ranges (parallel.cpp:21-29); the pick exchanges one record per
  // rank through an NCCL symmetric window (NVLink peer stores) and an LSA
  // barrier, then every rank commits the lexicographic minimum
  int rank, world, xch;
  ncclDevComm dcomm;
  ncclWindow_t win;
  int rec_bytes;              // per-rank record: {smice, index, key, pad, max_err[L]}
  int xemul;                  // > 1: one GPU plays xemul ranks (test aid, KRONRED_XCH_EMULATE)
  // complex objective (score_kernel<true>): super-node table of the active
  // list, each node's position in it, members of every super-node (CSR by
  // node id, kept in step with commit)
  int complex_obj;
  unsigned* snt;              // [n] (rho0 << 3) | mask per active super-node
  int* sn_pos;                // [n] position of an active super-node in sn
  int* mem_off;               // [n + 1]
  int* mem_list;              // [n]
  int* mem_tmp;               // [n] scratch of the member move
  volatile int* live_count;
  int* live_src;              // [cap][3]: s, r, candidate count
  double* live_smice;         // [cap]
  double* live_me;            // [cap][L]
  unsigned long long* live_t; // [cap] globaltimer at commit
};

constexpr unsigned kPadEntry = 7u;  // rho 0, first, phase 3 (inert row)
constexpr int kTabPadRows = 64;    // row-table padding >= largest scorer tile
constexpr int kLoopThreads = 1024;
constexpr int kIncCap = 512;  // incremental enumeration: largest removed / added key set

// first index in the ascending array v[0..n) whose value is >= x
__device__ __forceinline__ int lower_bound_u(const unsigned* v, int n, unsigned x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (v[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// 4-state transducer of the row-table layout: state q = rows mod 4 so far.
// A super-node with k rows that does not fit the current block is pushed to
// the next one (4 - q padding rows).
__device__ __forceinline__ void tab_step(int k, int& q, int& adv) {
  if (q + k > 4) {
    adv += 4 - q + k;
    q = k & 3;
  } else {
    adv += k;
    q = (q + k) & 3;
  }
}

// Composition of transducer maps over a chunk of super-nodes: for each start
// state s (rows mod 4 so far), the end state (2 bits each, packed) and the
// rows advanced. compose(A, B) = A then B.
struct TabMap {
  unsigned q;  // 4 x 2-bit end states
  int a0, a1, a2, a3;
};
__device__ __forceinline__ int tab_sel(const TabMap& m, unsigned s) {
  return s == 0u ? m.a0 : (s == 1u ? m.a1 : (s == 2u ? m.a2 : m.a3));
}
__device__ __forceinline__ TabMap tab_compose(const TabMap& A, const TabMap& B) {
  TabMap r;
  r.q = 0u;
  unsigned q1;
  q1 = A.q & 3u;
  r.q |= ((B.q >> (2u * q1)) & 3u);
  r.a0 = A.a0 + tab_sel(B, q1);
  q1 = (A.q >> 2) & 3u;
  r.q |= ((B.q >> (2u * q1)) & 3u) << 2;
  r.a1 = A.a1 + tab_sel(B, q1);
  q1 = (A.q >> 4) & 3u;
  r.q |= ((B.q >> (2u * q1)) & 3u) << 4;
  r.a2 = A.a2 + tab_sel(B, q1);
  q1 = (A.q >> 6) & 3u;
  r.q |= ((B.q >> (2u * q1)) & 3u) << 6;
  r.a3 = A.a3 + tab_sel(B, q1);
  return r;
}
__device__ __forceinline__ TabMap tab_shfl_up(const TabMap& m, int d) {
  TabMap r;
  r.q = __shfl_up_sync(0xffffffffu, m.q, d);
  r.a0 = __shfl_up_sync(0xffffffffu, m.a0, d);
  r.a1 = __shfl_up_sync(0xffffffffu, m.a1, d);
  r.a2 = __shfl_up_sync(0xffffffffu, m.a2, d);
  r.a3 = __shfl_up_sync(0xffffffffu, m.a3, d);
  return r;
}
// inclusive warp scan of maps (lane order = super-node order)
__device__ __forceinline__ TabMap tab_warp_scan(TabMap m, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const TabMap p = tab_shfl_up(m, d);
    if (lane >= d) m = tab_compose(p, m);
  }
  return m;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kLoopThreads) enum_kernel(LoopArgs a) {
  extern __shared__ unsigned keys[];  // [pow2 >= 2n]
  __shared__ int s_cnt;
  __shared__ TabMap wmap[kLoopThreads / 32];
  __shared__ int s_nrem, s_nnew;
  __shared__ int s_gbase[4], s_wcnt[kLoopThreads / 32][4];
  __shared__ unsigned s_rem[kIncCap], s_nk[kIncCap], s_remk[kIncCap];
  __shared__ unsigned long long gscan[kLoopThreads / 32];
  LoopState* st = a.st;
  const int tid = threadIdx.x;
  if (st->done) {
    if (a.use_cond && tid == 0) cudaGraphSetConditional(a.cond, 0u);
    return;
  }
  const int ns = st->ns;
  if (a.tdbg && tid == 0) a.tdbg[size_t(st->iter) * kTdbg + 2] = globaltimer();
  if (st->iter == 0 && tid == 0) {  // loop start: iteration 1's wall_ms
    const unsigned long long t = globaltimer();
    a.tr_t[a.cap] = t;
    if (a.live_count) *reinterpret_cast<volatile unsigned long long*>(a.live_count + 2) = t;
  }
#ifdef ENUM_TIMING
  long long et[9];
#endif

#ifdef ENUM_TIMING
  if (tid == 0) et[0] = clock64();
#endif
  if (a.complex_obj)  // complex scorer: active super-node table and positions
    for (int k = tid; k < ns; k += kLoopThreads) {
      const int i = a.sn[k];
      a.sn_pos[i] = k;
      a.snt[k] = (unsigned(a.prow_off[i]) << 3) | unsigned(a.mask[i]);
    }
  // ---- row table over the active super-nodes ------------------------------
  const int ch = (ns + kLoopThreads - 1) / kLoopThreads;
  const int b0 = min(ns, tid * ch), b1 = min(ns, b0 + ch);
  TabMap tmap;
  tmap.q = 0u;
  {
    int adv4[4];
#pragma unroll
    for (int q0 = 0; q0 < 4; ++q0) {
      int q = q0, adv = 0;
      for (int k = b0; k < b1; ++k) tab_step(__popc(a.mask[a.sn[k]]), q, adv);
      tmap.q |= unsigned(q) << (2 * q0);
      adv4[q0] = adv;
    }
    tmap.a0 = adv4[0];
    tmap.a1 = adv4[1];
    tmap.a2 = adv4[2];
    tmap.a3 = adv4[3];
  }
  // block scan of map composition (earlier map first): warp shuffles, the
  // warp totals scanned by warp 0, two barriers
#ifdef ENUM_TIMING
  if (tid == 0) et[1] = clock64();
#endif
  const int lane = tid & 31, warp = tid >> 5;
  const TabMap tincl = tab_warp_scan(tmap, lane);
  if (lane == 31) wmap[warp] = tincl;
  __syncthreads();
  if (warp == 0) wmap[lane] = tab_warp_scan(wmap[lane], lane);
  __syncthreads();
#ifdef ENUM_TIMING
  if (tid == 0) et[2] = clock64();
#endif
  {
    // state and table row entering this thread's chunk (from state 0 at row 0)
    int q = 0, t = 0;
    if (warp > 0) {
      const TabMap& w = wmap[warp - 1];
      q = int(w.q & 3u);
      t = w.a0;
    }
    const TabMap ex = tab_shfl_up(tincl, 1);
    if (lane > 0) {
      t += tab_sel(ex, unsigned(q));
      q = int((ex.q >> (2 * q)) & 3u);
    }
    for (int k = b0; k < b1; ++k) {
      const int i = a.sn[k];
      const unsigned m = a.mask[i];
      const int rows = __popc(m);
      if (q + rows > 4) {
        for (int u = q; u < 4; ++u) a.tab[t++] = kPadEntry;
        q = 0;
      }
      a.tab_of_node[i] = t;
      unsigned first = 4u;
      int rho = a.prow_off[i];
      for (int p = 0; p < 3; ++p)
        if ((m >> p) & 1u) {
          a.tab[t++] = (unsigned(rho++) << 3) | first | unsigned(p);
          first = 0u;
        }
      q = (q + rows) & 3;
    }
    if (tid == kLoopThreads - 1) {
      // tail: close the last block and add the scorer's tile padding
      const int tend = wmap[kLoopThreads / 32 - 1].a0;
      const int R = (tend + 3) & ~3;
      for (int u = tend; u < R + kTabPadRows; ++u) a.tab[u] = kPadEntry;
      st->R = R;
    }
  }

#ifdef ENUM_TIMING
  if (tid == 0) et[3] = clock64();
#endif
  // ---- candidates: super-node edges, both directions, filtered ------------
  if (a.tdbg && tid == 0) a.tdbg[size_t(st->iter) * kTdbg + 7] = globaltimer();
  // After a commit (s*, r*) only the keys with an end in {s*, r*} change: r*
  // is gone and s* owns the union of both edge sets (contracting a tree edge
  // creates no parallel edges, and the filters depend only on the two end
  // super-nodes). So the sorted list is the previous one minus those keys,
  // merged with the keys of s*'s edges re-generated from the branch list. A
  // full rebuild (generation + bitonic sort) runs on the first enumeration of
  // a reduction and whenever either change set exceeds kIncCap.
  const int C_old = st->C, ls = st->last_s, lr = st->last_r;
  bool inc = a.inc_enum && st->iter > 0 && C_old > 0;
  if (tid == 0) {
    s_cnt = 0;
    s_nrem = 0;
    s_nnew = 0;
  }
  __syncthreads();
  unsigned* old = keys + a.kcap;  // previous sorted keys (second region)
  if (inc) {
    for (int i = tid; i < C_old; i += kLoopThreads) {
      const int cs = a.cs[i], cr = a.cr[i];
      old[i] = (unsigned(cs) << 16) | unsigned(cr);
      if (cs == ls || cs == lr || cr == ls || cr == lr) {
        const int slot = atomicAdd(&s_nrem, 1);
        if (slot < kIncCap) s_rem[slot] = unsigned(i);
      }
    }
    for (int b = tid; b < a.nb; b += kLoopThreads) {
      const int x = a.sup[a.br_from[b]], y = a.sup[a.br_to[b]];
      if (x != y && (x == ls || y == ls)) {
        const unsigned mx = a.mask[x], my = a.mask[y];
        if (y != a.slack && (my & ~mx) == 0u) {
          const int slot = atomicAdd(&s_nnew, 1);
          if (slot < kIncCap) s_nk[slot] = (unsigned(x) << 16) | unsigned(y);
        }
        if (x != a.slack && (mx & ~my) == 0u) {
          const int slot = atomicAdd(&s_nnew, 1);
          if (slot < kIncCap) s_nk[slot] = (unsigned(y) << 16) | unsigned(x);
        }
      }
    }
    __syncthreads();
    inc = s_nrem <= kIncCap && s_nnew <= kIncCap;
  }
  int C;
  if (inc) {
    const int mr = s_nrem, mn = s_nnew;
    // rank sorts of the two small sets (values are unique)
    unsigned ri = 0u, nv = 0u;
    int rr = 0, rn = 0;
    if (tid < mr) {
      ri = s_rem[tid];
      for (int j = 0; j < mr; ++j) rr += s_rem[j] < ri ? 1 : 0;
    }
    if (tid < mn) {
      nv = s_nk[tid];
      for (int j = 0; j < mn; ++j) rn += s_nk[j] < nv ? 1 : 0;
    }
    __syncthreads();
    if (tid < mr) s_rem[rr] = ri;
    if (tid < mn) s_nk[rn] = nv;
    __syncthreads();
    if (tid < mr) s_remk[tid] = old[s_rem[tid]];  // removed keys, ascending
    __syncthreads();
    // kept key i lands at i - (removed before it) + (new keys below it);
    // new key j at (old keys below it) - (removed keys below it) + j
    for (int i = tid; i < C_old; i += kLoopThreads) {
      const unsigned k = old[i];
      const int cs = int(k >> 16), cr = int(k & 0xffffu);
      if (cs == ls || cs == lr || cr == ls || cr == lr) continue;
      keys[i - lower_bound_u(s_rem, mr, unsigned(i)) + lower_bound_u(s_nk, mn, k)] = k;
    }
    for (int j = tid; j < mn; j += kLoopThreads) {
      const unsigned v = s_nk[j];
      keys[lower_bound_u(old, C_old, v) - lower_bound_u(s_remk, mr, v) + j] = v;
    }
    C = C_old - mr + mn;
#ifdef ENUM_TIMING
    if (tid == 0) et[4] = et[5] = clock64();
#endif
    __syncthreads();
    if (C == 0) {
      if (tid == 0) {
        st->C = 0;
        st->done = 1;
        if (a.use_cond) cudaGraphSetConditional(a.cond, 0u);
      }
      return;
    }
  } else {
    // warp-aggregated slot allocation (one shared atomic per warp and direction)
    for (int b0 = 0; b0 < a.nb; b0 += kLoopThreads) {
      const int b = b0 + tid;
      bool e1 = false, e2 = false;
      unsigned k1 = 0, k2 = 0;
      if (b < a.nb) {
        const int x = a.sup[a.br_from[b]], y = a.sup[a.br_to[b]];
        if (x != y) {
          const unsigned mx = a.mask[x], my = a.mask[y];
          e1 = y != a.slack && (my & ~mx) == 0u;
          e2 = x != a.slack && (mx & ~my) == 0u;
          k1 = (unsigned(x) << 16) | unsigned(y);
          k2 = (unsigned(y) << 16) | unsigned(x);
        }
      }
      const unsigned lane_lt = (1u << (tid & 31)) - 1u;
      const unsigned m1 = __ballot_sync(0xffffffffu, e1), m2 = __ballot_sync(0xffffffffu, e2);
      const int n1 = __popc(m1), n2 = __popc(m2);
      int base = 0;
      if ((tid & 31) == 0 && n1 + n2 > 0) base = atomicAdd(&s_cnt, n1 + n2);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (e1) keys[base + __popc(m1 & lane_lt)] = k1;
      if (e2) keys[base + n1 + __popc(m2 & lane_lt)] = k2;
    }
#ifdef ENUM_TIMING
    if (tid == 0) et[4] = clock64();
#endif
    __syncthreads();
    C = s_cnt;
    if (C == 0) {
      if (tid == 0) {
        st->C = 0;
        st->done = 1;
        if (a.use_cond) cudaGraphSetConditional(a.cond, 0u);
      }
      return;
    }
    int N = 1;
    while (N < C) N <<= 1;
    for (int i = C + tid; i < N; i += kLoopThreads) keys[i] = 0xffffffffu;
    __syncthreads();
    for (int k = 2; k <= N; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < N; i += kLoopThreads) {
          const int l = i ^ j;
          if (l > i) {
            const unsigned ki = keys[i], kl = keys[l];
            const bool up = (i & k) == 0;
            if ((ki > kl) == up) {
              keys[i] = kl;
              keys[l] = ki;
            }
          }
        }
        __syncthreads();
      }
#ifdef ENUM_TIMING
    if (tid == 0) et[5] = clock64();
#endif
  }
  for (int i = tid; i < C; i += kLoopThreads) {
    a.cs[i] = int(keys[i] >> 16);
    a.cr[i] = int(keys[i] & 0xffffu);
  }

#ifdef ENUM_TIMING
  if (tid == 0) et[6] = clock64();
#endif
  // ---- group by |phi(r)| (stable) ----------------------------------------
  // Rounds of one element per thread (coalesced, independent loads): group
  // totals first (packed 3 x 21-bit counters, block reduction), then per
  // round a warp-ballot rank, a scan of the 32 warp counts and running group
  // bases.
  // this rank's contiguous range of the sorted list (parallel.cpp:21-29)
  const int xbase = C / a.world, xextra = C % a.world;
  const int c0 = a.rank * xbase + min(a.rank, xextra), Cl = xbase + (a.rank < xextra ? 1 : 0);
  unsigned long long mine = 0;
  for (int i = c0 + tid; i < c0 + Cl; i += kLoopThreads) mine += 1ull << (21 * (__popc(a.mask[keys[i] & 0xffffu]) - 1));
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if (lane == 0) gscan[warp] = mine;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = gscan[lane];
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (lane == 0) {
      const int c1 = int(w & 0x1fffff), c2 = int((w >> 21) & 0x1fffff);
      s_gbase[1] = 0;
      s_gbase[2] = c1;
      s_gbase[3] = c1 + c2;
    }
  }
  __syncthreads();
  const int cnt1 = s_gbase[2], cnt2 = s_gbase[3] - s_gbase[2];
  const unsigned lane_lt = (1u << lane) - 1u;
  for (int r0 = 0; r0 < Cl; r0 += kLoopThreads) {
    const int i = c0 + r0 + tid;  // global (lexicographic) index
    int s = 0, r = 0, g = 0;
    if (r0 + tid < Cl) {
      s = int(keys[i] >> 16);
      r = int(keys[i] & 0xffffu);
      g = __popc(a.mask[r]);
    }
    const unsigned b1 = __ballot_sync(0xffffffffu, g == 1), b2 = __ballot_sync(0xffffffffu, g == 2),
                   b3 = __ballot_sync(0xffffffffu, g == 3);
    if (lane == 0) {
      s_wcnt[warp][1] = __popc(b1);
      s_wcnt[warp][2] = __popc(b2);
      s_wcnt[warp][3] = __popc(b3);
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the warp counts, per group, plus the running base
#pragma unroll
      for (int gg = 1; gg <= 3; ++gg) {
        const int v = s_wcnt[lane][gg];
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        s_wcnt[lane][gg] = s_gbase[gg] + x - v;
        __syncwarp();
        if (lane == 31) s_gbase[gg] += x;
      }
    }
    __syncthreads();
    if (r0 + tid < Cl) {
      const unsigned bg = g == 1 ? b1 : (g == 2 ? b2 : b3);
      const int p = s_wcnt[warp][g] + __popc(bg & lane_lt);
      a.cand[p] = a.complex_obj ? make_int4(s, r, a.sn_pos[s], a.sn_pos[r])
                                : make_int4(s, r, a.tab_of_node[s], a.tab_of_node[r]);
      a.cidx[p] = i;
    }
    __syncthreads();  // s_wcnt is rewritten next round
  }
#ifdef ENUM_TIMING
  if (tid == 0) et[7] = clock64();
#endif
  // per 16-row scorer tile: plain (all first-of-super-node, no padding rows)
  {
    const int Rr = st->R;  // written by the last thread before the candidate section's barriers
    const int ntiles = (Rr + 15) / 16;
    for (int t = tid; t < ntiles; t += kLoopThreads) {
      unsigned all = 0xffffffffu, pad = 0u;
      for (int u = 0; u < 16; ++u) {
        const unsigned e = a.tab[16 * t + u];
        all &= e;
        pad |= e & (e >> 1) & 1u;  // phase 3
      }
      a.tplain[t] = (all & 4u) && !pad ? 1 : 0;
    }
  }
  if (tid == 0) {
    const int cnt3 = Cl - cnt1 - cnt2;
    const int S = s3_lanes((long long)Cl * a.L, a.fill, a.force_s, a.fill4_16);
    const int gk1 = a.gk1[S == 1 ? 0 : (S == 2 ? 1 : 2)];
    const int Sm = gk1 > 0 ? a.s_multi : S;  // split of the |phi(r)| >= 2 groups
    const int cpc1 = gk1 > 0 ? gk1 : s3_cpc(a.G3, 1, S), cpc2 = s3_cpc(a.G3, 2, Sm), cpc3 = s3_cpc(a.G3, 3, Sm);
    st->S = S;
    st->C = C;
    st->c0 = c0;
    st->Cl = Cl;
    if (a.use_scond) cudaGraphSetConditional(a.scond, S == 1 ? 0u : (S == 2 ? 1u : 2u));
    st->grp_start[0] = 0;
    st->grp_start[1] = 0;
    st->grp_start[2] = cnt1;
    st->grp_start[3] = cnt1 + cnt2;
    st->grp_cta[0] = 0;
    st->grp_cta[1] = (cnt1 + cpc1 - 1) / cpc1 * a.nsl;
    st->grp_cta[2] = st->grp_cta[1] + (cnt2 + cpc2 - 1) / cpc2 * a.nsl;
    st->grp_cta[3] = st->grp_cta[2] + (cnt3 + cpc3 - 1) / cpc3 * a.nsl;
    if (a.use_cond) cudaGraphSetConditional(a.cond, 1u);
    if (a.tdbg) a.tdbg[size_t(st->iter) * kTdbg + 3] = globaltimer();
#ifdef ENUM_TIMING
    et[8] = clock64();
    if (st->iter == 100 || st->iter == 500)
      printf("enum iter %d ns %d C %d: table pass1 %lld scan %lld emit %lld | keys %lld sort %lld out %lld group %lld tplain %lld\n",
             st->iter, ns, C, et[1] - et[0], et[2] - et[1], et[3] - et[2], et[4] - et[3], et[5] - et[4], et[6] - et[5],
             et[7] - et[6], et[8] - et[7]);
#endif
  }
}

__device__ __forceinline__ bool loop_better(double s1, int i1, double s2, int i2) {
  if (i1 < 0) return false;
  if (i2 < 0) return true;
  return s1 < s2 || (s1 == s2 && i1 < i2);
}

// first minimum feasible SMICE over candidates [lo, hi) (reduce.cpp:397-404),
// with its (s, r) key: thread strided scan, warp shuffles, then warp 0;
// every thread returns the block's result
__device__ __forceinline__ void pick_block_argmin(const LoopArgs& a, int lo, int hi, double* ss, int* si, unsigned* sk,
                                                  double& bs, int& bi, unsigned& bk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  bs = __longlong_as_double(0x7ff0000000000000LL);
  bi = -1;
  bk = 0u;
  for (int c = lo + tid; c < hi; c += kLoopThreads) {
    const double v = a.psm ? s3_candidate(a.psm, a.pmaxerr, c, a.L, a.ldc, a.e_bar) : a.pcand[c];
    const unsigned key = (unsigned(a.cs[c]) << 16) | unsigned(a.cr[c]);
    if (!(v < 0.0) && loop_better(v, c, bs, bi)) {
      bs = v;
      bi = c;
      bk = key;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double os = __shfl_down_sync(0xffffffffu, bs, o);
    const int oi = __shfl_down_sync(0xffffffffu, bi, o);
    const unsigned ok = __shfl_down_sync(0xffffffffu, bk, o);
    if (loop_better(os, oi, bs, bi)) {
      bs = os;
      bi = oi;
      bk = ok;
    }
  }
  __syncthreads();  // ss/si/sk may still be read from a previous call
  if (lane == 0) {
    ss[warp] = bs;
    si[warp] = bi;
    sk[warp] = bk;
  }
  __syncthreads();
  if (warp == 0) {
    bs = ss[lane];
    bi = si[lane];
    bk = sk[lane];
    for (int o = 16; o > 0; o >>= 1) {
      const double os = __shfl_down_sync(0xffffffffu, bs, o);
      const int oi = __shfl_down_sync(0xffffffffu, bi, o);
      const unsigned ok = __shfl_down_sync(0xffffffffu, bk, o);
      if (loop_better(os, oi, bs, bi)) {
        bs = os;
        bi = oi;
        bk = ok;
      }
    }
    if (lane == 0) {
      ss[0] = bs;
      si[0] = bi;
      sk[0] = bk;
    }
  }
  __syncthreads();
  bi = si[0];
  bs = ss[0];
  bk = sk[0];
}

__global__ void __launch_bounds__(kLoopThreads) pick_commit_kernel(LoopArgs a) {
  __shared__ double ss[32];
  __shared__ int si[32];
  __shared__ unsigned sk[32];
  __shared__ int s_pos;
  griddep_wait();
  // let the base refresh (the next kernel, launched programmatically) start
  // staging its constant program now; it waits for this grid before reading
  // anything the commit writes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  LoopState* st = a.st;
  if (st->done) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int C = st->C, c0 = st->c0, c1 = st->c0 + st->Cl;
  if (a.tdbg && tid == 0) a.tdbg[size_t(st->iter) * kTdbg + 0] = globaltimer();
#ifdef PICK_CLK  // timing experiment: SM cycles per pick phase (CTA thread 0)
  long long pk0 = clock64(), pk1 = 0, pk2 = 0, pk3 = 0;
#endif
  // the commit's first reads (super-node map and active list, which only this
  // kernel writes) are issued ahead of the argmin
  const int sup0 = tid < a.n ? a.sup[tid] : -1;
  const int sn0 = tid < st->ns ? a.sn[tid] : -1;
  // argmin with the candidate's (s, r) carried along (no dependent load after it)
  double bs;
  int bi;
  unsigned bk;
  pick_block_argmin(a, c0, c1, ss, si, sk, bs, bi, bk);
#ifdef PICK_CLK
  pk1 = clock64();
#endif
  const int L = a.L;
  const double* wme = nullptr;  // the winner's max_err[L] (its rank's record), else pmaxerr
  if (a.xch) {
    // min-loc over ranks: every rank stores its record {smice, index, key,
    // max_err[L]} into slot [parity][rank] of every rank's symmetric window
    // (NVLink stores), the LSA barrier orders them, and every rank merges the
    // same W records in rank order (lexicographic (smice, index); index < 0:
    // no feasible candidate on that rank). Slots alternate with the iteration
    // parity: a rank runs at most one barrier ahead of the slowest.
    // xemul > 1 (one GPU, test aid): this rank plays xemul ranks, each
    // reducing its own contiguous range into its own slot of the local window;
    // the merge below is the multi-rank one.
    const int par = st->iter & 1;
    const int W = a.xemul > 1 ? a.xemul : a.world;
    auto put = [&](char* dst, double vs, int vi, unsigned vk) {
      *reinterpret_cast<double*>(dst) = vs;
      *reinterpret_cast<long long*>(dst + 8) = vi;
      *reinterpret_cast<unsigned*>(dst + 16) = vk;
    };
    auto me_of = [&](int l, int idx) {
      return idx >= 0 ? (a.ldc > 0 ? a.pmaxerr[size_t(l) * a.ldc + idx] : a.pmaxerr[size_t(idx) * L + l]) : 0.0;
    };
    if (a.xemul > 1) {
      for (int q = 0; q < W; ++q) {
        const int xb = C / W, xe = C % W;
        const int lo = q * xb + min(q, xe), hi = lo + xb + (q < xe ? 1 : 0);
        double qs;
        int qi;
        unsigned qk;
        pick_block_argmin(a, lo, hi, ss, si, sk, qs, qi, qk);
        char* dst = static_cast<char*>(ncclGetLocalPointer(a.win, size_t(par * W + q) * a.rec_bytes));
        if (tid == 0) put(dst, qs, qi, qk);
        for (int l = tid; l < L; l += kLoopThreads) reinterpret_cast<double*>(dst + 24)[l] = me_of(l, qi);
        __syncthreads();
      }
    } else {
      const size_t my = size_t(par * W + a.rank) * size_t(a.rec_bytes);
      for (int q = tid; q < W; q += kLoopThreads) put(static_cast<char*>(ncclGetLsaPointer(a.win, my, q)), bs, bi, bk);
      for (int i = tid; i < W * L; i += kLoopThreads) {
        const int q = i / L, l = i - q * L;
        reinterpret_cast<double*>(static_cast<char*>(ncclGetLsaPointer(a.win, my, q)) + 24)[l] = me_of(l, bi);
      }
      ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), a.dcomm, ncclTeamLsa(a.dcomm), a.dcomm.lsaBarrier, 0);
      bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    }
    bs = __longlong_as_double(0x7ff0000000000000LL);
    bi = -1;
    bk = 0u;
    int wq = -1;
    for (int q = 0; q < W; ++q) {
      const char* src = static_cast<const char*>(ncclGetLocalPointer(a.win, size_t(par * W + q) * a.rec_bytes));
      const double qs = *reinterpret_cast<const volatile double*>(src);
      const long long qi = *reinterpret_cast<const volatile long long*>(src + 8);
      if (qi >= 0 && loop_better(qs, int(qi), bs, bi)) {
        bs = qs;
        bi = int(qi);
        bk = *reinterpret_cast<const volatile unsigned*>(src + 16);
        wq = q;
      }
    }
    if (wq >= 0)
      wme = reinterpret_cast<const double*>(
          static_cast<const char*>(ncclGetLocalPointer(a.win, size_t(par * W + wq) * a.rec_bytes)) + 24);
  }
  if (bi < 0) {  // no feasible assignment left (reduce.cpp:404)
    if (tid == 0) st->done = 1;
    return;
  }
  const int it = st->iter;
  const int s = int(bk >> 16), r = int(bk & 0xffffu);
  if (it < a.cap) {
    if (tid == 0) {
      a.tr_sr[2 * it] = s;
      a.tr_sr[2 * it + 1] = r;
      a.tr_c[it] = C;
      a.tr_smice[it] = bs;
      a.tr_t[it] = globaltimer();
    }
    for (int l = tid; l < L; l += kLoopThreads) {
      const double me = wme ? wme[l] : (a.ldc > 0 ? a.pmaxerr[size_t(l) * a.ldc + bi] : a.pmaxerr[size_t(bi) * L + l]);
      a.tr_me[size_t(it) * L + l] = me;
      if (a.live_count) a.live_me[size_t(it) * L + l] = me;
    }
    if (a.live_count && tid == 0) {
      a.live_src[3 * it] = s;
      a.live_src[3 * it + 1] = r;
      a.live_src[3 * it + 2] = C;
      a.live_smice[it] = bs;
      a.live_t[it] = globaltimer();
    }
  }
#ifdef PICK_CLK
  pk2 = clock64();
#endif
  // i_agg[s] += i_agg[r], i_agg[r] = 0 (reduce.cpp:336-343); bounds merge
  const unsigned ms = a.mask[s], mr = a.mask[r];
  const int rs0 = a.prow_off[s], rr0 = a.prow_off[r];
  for (int l = tid; l < L; l += kLoopThreads) {
    for (int p = 0; p < 3; ++p) {
      double2* ps = a.iagg + (size_t(s) * L + l) * 3 + p;
      double2* pr = a.iagg + (size_t(r) * L + l) * 3 + p;
      const C2 sum = dev::cadd(ld2(ps), ld2(pr));
      st2(ps, sum);
      *pr = make_double2(0.0, 0.0);
      if ((ms >> p) & 1u) st2(a.iaggp + size_t(l) * a.nphi + rs0 + popc_below(ms, p), sum);
      if ((mr >> p) & 1u) {
        a.iaggp[size_t(l) * a.nphi + rr0 + popc_below(mr, p)] = make_double2(0.0, 0.0);
        double2* dst = a.bv + bv_bnd(size_t(rs0 + popc_below(ms, p)), L, l);
        const double2 bb = a.bv[bv_bnd(size_t(rr0 + popc_below(mr, p)), L, l)];
        const double2 cur = *dst;
        *dst = make_double2(dmin(cur.x, bb.x), dmax(cur.y, bb.y));
      }
    }
  }
  for (int j = tid; j < a.n; j += kLoopThreads)
    if ((j == tid ? sup0 : a.sup[j]) == r) a.sup[j] = s;
  if (a.complex_obj) {
    // members: r's list joins the end of s's (reduce.cpp:326-329 append
    // order), the lists between the two move by |members(r)|
    const int os0 = a.mem_off[s], os1 = a.mem_off[s + 1], or0 = a.mem_off[r], or1 = a.mem_off[r + 1];
    const int kr = or1 - or0;
    const int A = s < r ? os1 : or0, B = s < r ? or1 : os1;
    for (int x = A + tid; x < B; x += kLoopThreads) {
      int src;
      if (s < r)  // [r's members][lists s+1 .. r-1]
        src = x - A < kr ? or0 + (x - A) : x - kr;
      else  // [lists r+1 .. s][r's members]
        src = x < B - kr ? x + kr : or0 + (x - (B - kr));
      a.mem_tmp[x] = a.mem_list[src];
    }
    __syncthreads();
    for (int x = A + tid; x < B; x += kLoopThreads) a.mem_list[x] = a.mem_tmp[x];
    if (s < r)
      for (int i = s + 1 + tid; i <= r; i += kLoopThreads) a.mem_off[i] += kr;
    else
      for (int i = r + 1 + tid; i <= s; i += kLoopThreads) a.mem_off[i] -= kr;
    (void)os0;
  }
#ifdef PICK_CLK
  pk3 = clock64();
#endif
  // remove r from the ascending active list
  const int ns = st->ns;
  for (int k = tid; k < ns; k += kLoopThreads)
    if ((k == tid ? sn0 : a.sn[k]) == r) s_pos = k;
  __syncthreads();
  // shift the tail left by one, a block-wide chunk at a time (each chunk is
  // read completely before any of it is written)
  for (int base = s_pos + 1; base < ns; base += kLoopThreads) {
    const int k = base + tid;
    const int v = k < ns ? a.sn[k] : 0;
    __syncthreads();
    if (k < ns) a.sn[k - 1] = v;
    __syncthreads();
  }
  if (tid == 0) {
    st->ns = ns - 1;
    st->iter = it + 1;
    st->last_s = s;
    st->last_r = r;
    if (a.has_target && double(a.n - (ns - 1)) / double(a.n) >= a.target) st->done = 1;
    if (it + 1 >= a.cap) st->done = 1;
    if (a.tdbg) a.tdbg[size_t(it) * kTdbg + 1] = globaltimer();
#ifdef PICK_CLK
    if (a.tdbg) {
      const long long pk4 = clock64();
      a.tdbg[size_t(it) * kTdbg + 12] = (unsigned long long)((pk1 - pk0) | ((pk2 - pk1) << 16) | ((pk3 - pk2) << 32) | ((pk4 - pk3) << 48));
    }
#endif
    if (a.live_count && it < a.cap) {
      // every thread's row stores precede the barriers above; make them
      // visible to the host before the count that publishes the row
      __threadfence_system();
      *a.live_count = it + 1;
    }
  }
}

}  // namespace
}  // namespace kronred::b200
