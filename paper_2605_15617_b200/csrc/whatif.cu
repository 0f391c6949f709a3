// whatif.cu — rows f1, f3, f4 on the replay engine: per-node durations / memory deltas and the
// critical path.
//
//  * f1 inter-slice calibration (§5.3): the timed graph filled slice by slice (each
//    rank's nodes measured while it ran as a real rank) is re-timed by the same ASAP replay, which
//    "shift[s] the receive to occur after the send" and propagates; the input is one measured
//    duration per node.
//  * f3 what-if ("a fake GPU kernel that spins for the desired and optimized
//    duration"; SPEC S:488-505 what_if / fault_inject): label overrides and per-rank compute
//    slowdown (P:1751-1760 thermal throttling), then the critical path that decides T.
//  * f4 MoE imbalance (P:1745-1748 mock router): per-(stage, ep-rank) expert / all-to-all
//    durations and activation sizes arrive as per-node durations and memory deltas.
// Effective duration of node n: base (measured, else template) -> label override -> (d * f_r) >> 16
// for compute spans of rank r. A synchronization group lasts the max of its members' effective
// durations (reading Z2). The replay kernels read these through pointer-swapped DevGraph arrays.
#include <cuda_runtime.h>

#include "graph.h"

namespace prism {

namespace {

constexpr uint64_t K_GOLD = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t K_MIX = 0xBF58476D1CE4E5B9ULL;

// Effective per-node durations and memory deltas (rows f1/f3/f4), one thread per node n of rank r
// running template op ti of its stage:
//   d = measured (in.base[n]) else template;  d = (d * br) >> 16 if op ti is routed by gating event
//   v (MoE mock router: br[v][ep_i(r)] = the rank's share of event v's tokens
//   relative to the uniform share, Q16);  d = label_dur[i] if label(n) == labels[i];
//   d = (d * rank_f[r]) >> 16 for compute spans (fault injection).
//   alloc / free = given (in.al / in.fr) else template, then scaled by br like d (scale bits).
// Out-of-range inputs set *status (validation runs here, not in an O(N) host loop).
__global__ void __launch_bounds__(256) eff_kernel(DevGraph g, DurIn in, MoeIn me, int64_t *__restrict__ eff,
                                                  int64_t *__restrict__ eal, int64_t *__restrict__ efr,
                                                  uint32_t *status) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < g.N; n += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = in.base ? in.base[n] : nd_dur(g, (int32_t)n);
    if (d < 0 || d > (1LL << 40)) atomicCAS(status, 0u, (uint32_t)PRISM_E_INVALID_ARG);
    const int32_t r = g.node_rank[n];
    int32_t b = 65536;  // br of the node's gating event on its EP rank (Q16), 1.0 if not routed
    if (me.n_events > 0) {
      const int32_t s = g.rank_stage[r];
      const int64_t ti = g.t_op0[s] + (n - g.rank_ptr[r]);
      const int32_t v = me.op_event[ti];
      if (v >= 0) {
        const int32_t dpi = g.order == PRISM_ORDER_MEGATRON ? (r / g.tp) % g.dp : r / (g.tp * g.pp);
        b = me.br[(int64_t)v * g.ep + dpi % g.ep];
      }
    }
    if (me.scale & PRISM_MOE_DUR) d = (d * (int64_t)b) >> 16;
    if (in.n_labels > 0) {
      const uint32_t L = nd_label(g, (int32_t)n);
      int32_t lo = 0, hi = in.n_labels - 1;
      while (lo <= hi) {
        const int32_t mid = (lo + hi) >> 1;
        const uint32_t v = in.labels[mid];
        if (v == L) {
          d = in.label_dur[mid];
          break;
        }
        if (v < L) lo = mid + 1;
        else hi = mid - 1;
      }
    }
    if (in.rank_f && nd_kind(g, (int32_t)n) == PRISM_KIND_COMPUTE) d = (d * (int64_t)in.rank_f[r]) >> 16;
    eff[n] = d;
    if (eal) {
      int64_t a = in.al ? in.al[n] : nd_alloc(g, (int32_t)n), f = in.fr ? in.fr[n] : nd_free(g, (int32_t)n);
      if (a < 0 || f < 0 || a > (1LL << 43) || f > (1LL << 43)) atomicCAS(status, 0u, (uint32_t)PRISM_E_INVALID_ARG);
      if (me.scale & PRISM_MOE_ALLOC) a = (a * (int64_t)b) >> 16;
      if (me.scale & PRISM_MOE_FREE) f = (f * (int64_t)b) >> 16;
      eal[n] = a;
      efr[n] = f;
    }
  }
}

// The running allocation of every rank never drops below zero (program order, reading Z6): one
// warp per rank, 64-bit warp scan of (alloc - free) with the running minimum per lane.
__global__ void __launch_bounds__(256) mem_check_kernel(DevGraph g, const int64_t *__restrict__ al,
                                                        const int64_t *__restrict__ fr, uint32_t *status) {
  const int lane = threadIdx.x & 31;
  const int32_t warps = gridDim.x * (blockDim.x >> 5);
  for (int32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < g.W; r += warps) {
    const int32_t rb = g.rank_ptr[r], re = g.rank_ptr[r + 1];
    int64_t carry = 0;
    bool neg = false;
    for (int32_t base = rb; base < re; base += 32) {
      const int32_t i = base + lane;
      int64_t x = i < re ? al[i] - fr[i] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      neg |= i < re && carry + x < 0;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (__any_sync(0xffffffffu, neg) && lane == 0) atomicCAS(status, 0u, (uint32_t)PRISM_E_NEGATIVE_MEMORY);
  }
}

// Group durations = max over members' effective durations (Z2); then the per-node replay record
// (compute: own; sync: its first group's) and the per-slot record of the cell kernel.
__global__ void __launch_bounds__(256) grp_dur_kernel(DevGraph g, const int64_t *__restrict__ eff,
                                                      int64_t *__restrict__ gdur) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < g.G; x += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = 0;
    for (int32_t j = g.grp_ptr[x]; j < g.grp_ptr[x + 1]; ++j) m = max(m, eff[g.grp_mem[j]]);
    gdur[x] = m;
  }
}

__global__ void __launch_bounds__(256) records_kernel(DevGraph g, const int64_t *__restrict__ eff,
                                                      const int64_t *__restrict__ gdur,
                                                      int64_t *__restrict__ sdur, int64_t *__restrict__ hdur) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < g.N; n += stride) {
    const int32_t h0 = g.node_gptr[n], h1 = g.node_gptr[n + 1];
    sdur[n] = h0 == h1 ? eff[n] : gdur[g.node_grp[h0]];
  }
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < g.M; h += stride) hdur[h] = gdur[g.node_grp[h]];
}


// Row f3, step 0: T_k = max over every node's finish (covers multi-stream ranks, whose last op in
// issue order need not finish last).
__global__ void __launch_bounds__(256) view_max_kernel(DevGraph g, const int64_t *__restrict__ fin, int32_t Sp,
                                                       int32_t k, int64_t *__restrict__ T) {
  int64_t m = 0;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < g.N; n += (int64_t)gridDim.x * blockDim.x)
    m = max(m, fin[fin_off(g, fin_row(g, (int32_t)n), k, Sp)]);
  for (int off = 16; off; off >>= 1) m = max(m, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)m, off));
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long *)T, (unsigned long long)m);
}

// Row f3, step 1: T_k and the lowest node finishing at T_k.
__global__ void __launch_bounds__(256) crit_start_kernel(DevGraph g, const int64_t *__restrict__ fin,
                                                         int32_t Sp, int32_t k, const int64_t *__restrict__ iter,
                                                         int32_t *__restrict__ out_node) {
  const int64_t T = iter[k];
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < g.N; n += (int64_t)gridDim.x * blockDim.x)
    if (fin[fin_off(g, fin_row(g, (int32_t)n), k, Sp)] == T) atomicMin(out_node, (int32_t)n);
}

// Row f3, steps 2-4. The walk's rules are the oracle's (oracle/prism_oracle.cpp
// oracle_critical_path, reading R6): compute span <- its directional predecessor; sync node <- its
// group with the max (start + dur') (lowest uid on ties) <- that group's latest-ready member (lowest
// node id on ties) <- the member's directional predecessor; the walk ends at a node without one.
// Every choice depends only on the recorded times, so the parent of EVERY node is computed in
// parallel (groups first, then nodes) and the walk is a chase through the parent array (held in
// L2) instead of a serial scan of each group's members.
//
// A node's directional predecessor: its stream predecessor (row f2: or its event source,
// whichever finished later, the lower id on ties).
__device__ __forceinline__ int32_t crit_pred(const DevGraph &g, const int64_t *fin, int32_t Sp, int32_t k, int32_t n) {
  if (!g.ms) return g.rank_ptr[g.node_rank[n]] == n ? -1 : n - 1;
  const int32_t a = g.node_spred[n], b = g.node_esrc[n];
  if (a < 0) return b;
  if (b < 0) return a;
  const int64_t fa = fin[fin_off(g, fin_row(g, a), k, Sp)], fb = fin[fin_off(g, fin_row(g, b), k, Sp)];
  if (fa != fb) return fa > fb ? a : b;
  return min(a, b);
}

// step 2: per group (one warp), start = max over members of ready(member) and the latest-ready
// member (lowest node id on ties)
__global__ void __launch_bounds__(256) crit_groups_kernel(DevGraph g, const int64_t *__restrict__ fin, int32_t Sp,
                                                          int32_t k, int64_t *__restrict__ gstart,
                                                          int32_t *__restrict__ gbest) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t gi = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); gi < g.G; gi += warps) {
    int64_t br = -1;
    int32_t bm = 0x7FFFFFFF;
    for (int32_t j = g.grp_ptr[gi] + lane; j < g.grp_ptr[gi + 1]; j += 32) {
      const int32_t m = g.grp_mem[j];
      const int32_t q = crit_pred(g, fin, Sp, k, m);
      const int64_t r = q < 0 ? 0 : fin[fin_off(g, fin_row(g, q), k, Sp)];
      if (r > br || (r == br && m < bm)) {
        br = r;
        bm = m;
      }
    }
    for (int off = 16; off; off >>= 1) {
      const int64_t r2 = (int64_t)__shfl_xor_sync(0xffffffffu, (long long)br, off);
      const int32_t m2 = __shfl_xor_sync(0xffffffffu, bm, off);
      if (r2 > br || (r2 == br && m2 < bm)) {
        br = r2;
        bm = m2;
      }
    }
    if (lane == 0) {
      gstart[gi] = br;
      gbest[gi] = bm;
    }
  }
}

// step 3: the parent of every node (-1: none)
__global__ void __launch_bounds__(256) crit_parent_kernel(DevGraph g, ScenParams p, const int64_t *__restrict__ fin,
                                                          int32_t Sp, int32_t k, const int64_t *__restrict__ gstart,
                                                          const int32_t *__restrict__ gbest, int32_t *__restrict__ parent) {
  const int32_t kg = p.first + k;  // global scenario index (perturbation key)
  for (int64_t nn = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; nn < g.N; nn += (int64_t)gridDim.x * blockDim.x) {
    const int32_t n = (int32_t)nn;
    const int32_t h0 = g.node_gptr[n], h1 = g.node_gptr[n + 1];
    if (h0 == h1) {
      parent[n] = crit_pred(g, fin, Sp, k, n);
      continue;
    }
    int64_t bf = -1;
    uint64_t buid = 0;
    int32_t bg = -1;
    for (int32_t h = h0; h < h1; ++h) {
      const int32_t gi = g.node_grp[h];
      const uint64_t uid = g.grp_uid[gi];
      const uint32_t gb = (uid >> 56) == PRISM_ROLE_P2P ? 4u : 2u;
      int64_t d = g.grp_dur[gi];
      if ((p.mask & gb) && p.amp > 0 && kg > 0) d = perturb_x(d, p.seed ^ ((uint64_t)kg * K_GOLD) ^ (uid * K_MIX), p);
      const int64_t f = gstart[gi] + d;
      if (f > bf || (f == bf && uid < buid)) {
        bf = f;
        buid = uid;
        bg = gi;
      }
    }
    parent[n] = crit_pred(g, fin, Sp, k, gbest[bg]);
  }
}

// step 4: runs of stream predecessors. Inside a rank, a node whose parent is the node before it
// continues the run of that node; run_start[n] = the first node of n's run (a warp per rank:
// prefix max of the run-break positions), so the chase below needs two dependent loads per RUN
// (one per hop between ranks / groups) instead of one per node.
__global__ void __launch_bounds__(256) crit_runs_kernel(DevGraph g, const int32_t *__restrict__ parent,
                                                        int2 *__restrict__ run) {
  const int lane = threadIdx.x & 31;
  const int32_t warps = gridDim.x * (blockDim.x >> 5);
  for (int32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < g.W; r += warps) {
    const int32_t rb = g.rank_ptr[r], re = g.rank_ptr[r + 1];
    int32_t carry = rb;
    for (int32_t base = rb; base < re; base += 32) {
      const int32_t i = base + lane;
      int32_t x = (i < re && (i == rb || parent[i] != i - 1)) ? i : carry;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) x = max(x, __shfl_up_sync(0xffffffffu, x, off));
      x = max(x, carry);
      if (i < re) run[i] = make_int2(x, parent[x]);  // the run's first node and where it leads
      carry = __shfl_sync(0xffffffffu, x, 31);
    }
  }
}

// step 5: the chase from the lowest node finishing at T (one thread): one dependent 8-byte load per
// run (its first node and that node's parent), the run itself written out without loads
__global__ void crit_chase_kernel(const int32_t *__restrict__ start_node, int32_t N, const int2 *__restrict__ run,
                                  int32_t *__restrict__ path, int64_t cap, int64_t *__restrict__ len_out) {
  int32_t cur = *start_node;
  if (cur < 0 || cur >= N) cur = -1;  // empty graph: empty path
  int64_t len = 0;
  while (cur >= 0) {
    const int2 rn = __ldcg(run + cur);
    const int32_t rs = rn.x, nxt = rn.y;
    for (int32_t x = cur; x >= rs; --x, ++len)
      if (len < cap) path[len] = x;
    cur = nxt;
  }
  *len_out = len;
}

}  // namespace

cudaError_t launch_durations(const DevGraph &g, const DurIn &in, const MoeIn &me, int64_t *eff, int64_t *eal,
                             int64_t *efr, int64_t *gdur, int64_t *sdur, int64_t *hdur, uint32_t *status,
                             cudaStream_t st) {
  const int blocks = num_sms() * 8;
  if (g.N > 0) eff_kernel<<<blocks, 256, 0, st>>>(g, in, me, eff, eal, efr, status);
  if (eal && g.W > 0) mem_check_kernel<<<blocks, 256, 0, st>>>(g, eal, efr, status);
  if (g.G > 0) grp_dur_kernel<<<blocks, 256, 0, st>>>(g, eff, gdur);
  if (g.N > 0 || g.M > 0) records_kernel<<<blocks, 256, 0, st>>>(g, eff, gdur, sdur, hdur);
  return cudaGetLastError();
}

cudaError_t launch_critical_path(const DevGraph &g, const ScenParams &p, const int64_t *fin, int32_t Sp, int32_t k,
                                 int64_t *iter, int32_t *scratch, int32_t *path, int64_t cap, int64_t *len_out,
                                 int64_t *gstart, int32_t *gbest, int32_t *parent, int32_t *run_start,
                                 bool have_T, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(scratch, 0x7F, 4, st);
  if (e == cudaSuccess && !have_T) e = cudaMemsetAsync(iter + k, 0, 8, st);
  if (e != cudaSuccess) return e;
  const int blocks = num_sms() * 8;
  if (g.N > 0 && !have_T) view_max_kernel<<<blocks, 256, 0, st>>>(g, fin, Sp, k, iter + k);
  if (g.N > 0) crit_start_kernel<<<blocks, 256, 0, st>>>(g, fin, Sp, k, iter, scratch);
  if (g.G > 0) crit_groups_kernel<<<blocks, 256, 0, st>>>(g, fin, Sp, k, gstart, gbest);
  if (g.N > 0) crit_parent_kernel<<<blocks, 256, 0, st>>>(g, p, fin, Sp, k, gstart, gbest, parent);
  int2 *run = reinterpret_cast<int2 *>(run_start);  // 8-byte aligned scratch of 2 N words
  if (g.W > 0) crit_runs_kernel<<<blocks, 256, 0, st>>>(g, parent, run);
  crit_chase_kernel<<<1, 1, 0, st>>>(scratch, (int32_t)g.N, run, path, cap, len_out);
  return cudaGetLastError();
}

}  // namespace prism
