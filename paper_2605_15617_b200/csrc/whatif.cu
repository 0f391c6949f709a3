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


// Row f3, step 0 (sharded views; the unsharded replay reduces its rank ends instead): T_k = max
// over every node's finish. A single-stream rank's finish times never decrease along its stream, so
// its last node finishes last (a thread per rank); multi-stream ranks scan every node.
__global__ void __launch_bounds__(256) view_max_kernel(DevGraph g, const int64_t *__restrict__ fin, int32_t Sp,
                                                       int32_t k, int64_t *__restrict__ T) {
  int64_t m = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (g.ms) {
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < g.N; n += stride)
      m = max(m, fin[fin_off(g, fin_row(g, (int32_t)n), k, Sp)]);
  } else {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < g.W; r += stride) {
      const int32_t rb = g.rank_ptr[r], re = g.rank_ptr[r + 1];
      if (re > rb)
        m = max(m, fin[fin_off(g, cell_row0(g, (int32_t)r) + (int64_t)(re - 1 - rb) * cell_row_stride(g), k, Sp)]);
    }
  }
  for (int off = 16; off; off >>= 1) m = max(m, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)m, off));
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long *)T, (unsigned long long)m);
}

// Row f3, step 1: the lowest node finishing at T_k. Multi-stream graphs: every node is compared.
// Single-stream: a warp per rank; only a rank whose last node finishes at T_k holds such nodes, as
// a suffix (finish times never decrease along the stream), whose first node is found scanning back.
__global__ void __launch_bounds__(256) crit_start_kernel(DevGraph g, const int64_t *__restrict__ fin,
                                                         int32_t Sp, int32_t k, const int64_t *__restrict__ iter,
                                                         int32_t *__restrict__ out_node) {
  const int64_t T = iter[k];
  if (g.ms) {
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < g.N; n += (int64_t)gridDim.x * blockDim.x)
      if (fin[fin_off(g, fin_row(g, (int32_t)n), k, Sp)] == T) atomicMin(out_node, (int32_t)n);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int32_t warps = gridDim.x * (blockDim.x >> 5);
  const int32_t cs = cell_row_stride(g);
  for (int32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < g.W; r += warps) {
    const int32_t rb = g.rank_ptr[r], re = g.rank_ptr[r + 1];
    if (re == rb) continue;
    const int64_t row0 = cell_row0(g, r);
    if (fin[fin_off(g, row0 + (int64_t)(re - 1 - rb) * cs, k, Sp)] != T) continue;
    int32_t lo = rb;
    for (int32_t top = re; top > rb; top -= 32) {
      const int32_t i = top - 32 + lane;
      const bool below = i >= rb && fin[fin_off(g, row0 + (int64_t)(i - rb) * cs, k, Sp)] != T;
      const uint32_t bal = __ballot_sync(0xffffffffu, below);
      if (bal) {
        lo = top - 32 + (31 - __clz(bal)) + 1;
        break;
      }
    }
    if (lane == 0) atomicMin(out_node, lo);
  }
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
// A member's ready time: its directional predecessor's finish (0 without one).
__device__ __forceinline__ int64_t crit_ready(const DevGraph &g, const int64_t *fin, int32_t Sp, int32_t k,
                                              int32_t n) {
  if (g.ms) {
    const int32_t q = crit_pred(g, fin, Sp, k, n);
    return q < 0 ? 0 : fin[fin_off(g, fin_row(g, q), k, Sp)];
  }
  const int32_t r = g.node_rank[n], rb = g.rank_ptr[r];
  return n == rb ? 0 : fin[fin_off(g, cell_row0(g, r) + (int64_t)(n - 1 - rb) * cell_row_stride(g), k, Sp)];
}
// Groups' (start, latest-ready member) as one 64-bit max key: ready << 25 | (2^25 - 1 - member),
// so the max is the latest ready time and, among equals, the lowest member; it needs N < 2^25 and
// T < 2^38 (every ready time is <= T). Otherwise the key is the ready time alone and a second pass
// takes the lowest member at that time.
__device__ __forceinline__ bool crit_packed(const DevGraph &g, int64_t T) {
  return g.N < (1LL << 25) && T < (1LL << 38);
}

// step 2a: a thread per node; each sync node max-es its ready key into each of its groups
__global__ void __launch_bounds__(256) crit_ready_kernel(DevGraph g, const int64_t *__restrict__ fin, int32_t Sp,
                                                         int32_t k, const int64_t *__restrict__ iter,
                                                         int64_t *__restrict__ gkey) {
  const bool packed = crit_packed(g, iter[k]);
  for (int64_t nn = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; nn < g.N; nn += (int64_t)gridDim.x * blockDim.x) {
    const int32_t n = (int32_t)nn;
    const int32_t h0 = g.node_gptr[n], h1 = g.node_gptr[n + 1];
    if (h0 == h1) continue;
    const int64_t r = crit_ready(g, fin, Sp, k, n);
    const int64_t key = packed ? (r << 25) | (int64_t)(0x1FFFFFF - n) : r;
    for (int32_t h = h0; h < h1; ++h) atomicMax((unsigned long long *)(gkey + g.node_grp[h]), (unsigned long long)key);
  }
}

// step 2b (unpacked keys only): the lowest member whose ready time is its group's start
__global__ void __launch_bounds__(256) crit_tie_kernel(DevGraph g, const int64_t *__restrict__ fin, int32_t Sp,
                                                       int32_t k, const int64_t *__restrict__ iter,
                                                       const int64_t *__restrict__ gkey, int32_t *__restrict__ gbest) {
  if (crit_packed(g, iter[k])) return;
  for (int64_t nn = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; nn < g.N; nn += (int64_t)gridDim.x * blockDim.x) {
    const int32_t n = (int32_t)nn;
    const int32_t h0 = g.node_gptr[n], h1 = g.node_gptr[n + 1];
    if (h0 == h1) continue;
    const int64_t r = crit_ready(g, fin, Sp, k, n);
    for (int32_t h = h0; h < h1; ++h) {
      const int32_t gi = g.node_grp[h];
      if (gkey[gi] == r) atomicMin(gbest + gi, n);
    }
  }
}

// step 3a: a thread per group: its finish start + dur' (in place of the key) and the parent its
// sync nodes take if it is their latest group (in place of the best member), which the chase may
// jump to: marked in the target bitmap tgt
__global__ void __launch_bounds__(256) crit_gfin_kernel(DevGraph g, ScenParams p, const int64_t *__restrict__ fin,
                                                        int32_t Sp, int32_t k, const int64_t *__restrict__ iter,
                                                        int64_t *__restrict__ gkey, int32_t *__restrict__ gbest,
                                                        uint32_t *__restrict__ tgt) {
  const bool packed = crit_packed(g, iter[k]);
  const int32_t kg = p.first + k;  // global scenario index (perturbation key)
  for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < g.G; gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t key = gkey[gi];
    const int64_t start = packed ? key >> 25 : key;
    const int32_t best = packed ? (key == 0 ? -1 : 0x1FFFFFF - (int32_t)(key & 0x1FFFFFF)) : gbest[gi];
    if (best < 0 || best >= g.N) {  // an instance no node joins (G counts every instance of a quotient group)
      gbest[gi] = -1;
      continue;
    }
    const uint64_t uid = g.grp_uid[gi];
    const uint32_t gb = (uid >> 56) == PRISM_ROLE_P2P ? 4u : 2u;
    int64_t d = g.grp_dur[gi];
    if ((p.mask & gb) && p.amp > 0 && kg > 0) d = perturb_x(d, p.seed ^ ((uint64_t)kg * K_GOLD) ^ (uid * K_MIX), p);
    gkey[gi] = start + d;
    const int32_t t = crit_pred(g, fin, Sp, k, best);
    gbest[gi] = t;
    if (t >= 0) atomicOr(tgt + (t >> 5), 1u << (t & 31));
  }
}

// step 3b: the parent of every node (-1: none); jump targets other than groups' parents (the
// start node, multi-stream event sources) are marked in tgt
__global__ void __launch_bounds__(256) crit_parent_kernel(DevGraph g, const int64_t *__restrict__ fin, int32_t Sp,
                                                          int32_t k, const int64_t *__restrict__ gfin,
                                                          const int32_t *__restrict__ gpar, int32_t *__restrict__ parent,
                                                          const int32_t *__restrict__ start_node,
                                                          uint32_t *__restrict__ tgt) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int32_t s = *start_node;
    if (s >= 0 && s < g.N) atomicOr(tgt + (s >> 5), 1u << (s & 31));
  }
  for (int64_t nn = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; nn < g.N; nn += (int64_t)gridDim.x * blockDim.x) {
    const int32_t n = (int32_t)nn;
    const int32_t h0 = g.node_gptr[n], h1 = g.node_gptr[n + 1];
    if (h0 == h1) {
      const int32_t q = crit_pred(g, fin, Sp, k, n);
      parent[n] = q;
      if (g.ms && q >= 0 && q != n - 1) atomicOr(tgt + (q >> 5), 1u << (q & 31));
      continue;
    }
    int32_t bg = g.node_grp[h0];
    int64_t bf = gfin[bg];
    for (int32_t h = h0 + 1; h < h1; ++h) {
      const int32_t gi = g.node_grp[h];
      const int64_t f = gfin[gi];
      if (f > bf || (f == bf && g.grp_uid[gi] < g.grp_uid[bg])) {
        bf = f;
        bg = gi;
      }
    }
    parent[n] = gpar[bg];
  }
}

// step 4: the jump targets (nodes the chase can land on) are numbered in node order: a prefix sum
// of the target bitmap's popcounts (kScanWords words per block: block sums, then each block's
// offset and its words' prefixes).
constexpr int kScanWords = 2048;
__global__ void __launch_bounds__(256) crit_bsum_kernel(const uint32_t *__restrict__ tgt, int64_t nw,
                                                        int32_t *__restrict__ bsum) {
  __shared__ int32_t part[8];
  const int64_t w0 = (int64_t)blockIdx.x * kScanWords;
  int32_t c = 0;
  for (int64_t w = w0 + threadIdx.x; w < min(w0 + (int64_t)kScanWords, nw); w += blockDim.x) c += __popc(tgt[w]);
  for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t t = 0;
    for (int i = 0; i < 8; ++i) t += part[i];
    bsum[blockIdx.x] = t;
  }
}
// wpre[w] = targets in words < w (8 consecutive words per thread, block-wide exclusive scan)
__global__ void __launch_bounds__(256) crit_wpre_kernel(const uint32_t *__restrict__ tgt, int64_t nw,
                                                        const int32_t *__restrict__ bsum, int32_t *__restrict__ wpre) {
  __shared__ int32_t warp_tot[8];
  __shared__ int32_t base_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x < 32) {  // this block's offset: the sum of the earlier blocks' counts
    int32_t b = 0;
    for (int i = lane; i < (int)blockIdx.x; i += 32) b += bsum[i];
    for (int off = 16; off; off >>= 1) b += __shfl_xor_sync(0xffffffffu, b, off);
    if (lane == 0) base_s = b;
  }
  const int64_t w0 = (int64_t)blockIdx.x * kScanWords + threadIdx.x * 8;
  int32_t c[8], tot = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c[i] = w0 + i < nw ? __popc(tgt[w0 + i]) : 0;
    tot += c[i];
  }
  int32_t inc = tot;
  for (int off = 1; off < 32; off <<= 1) {
    const int32_t v = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += v;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  int32_t pre = base_s + inc - tot;
  for (int i = 0; i < wid; ++i) pre += warp_tot[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (w0 + i < nw) wpre[w0 + i] = pre;
    pre += c[i];
  }
}
__device__ __forceinline__ int32_t crit_tidx(const uint32_t *tgt, const int32_t *wpre, int32_t t) {
  return wpre[t >> 5] + __popc(tgt[t >> 5] & ((1u << (t & 31)) - 1u));
}

// step 5: runs of stream predecessors. Inside a rank, a node whose parent is the node before it
// continues the run of that node; the first node of each node's run is a prefix max of the
// run-break positions (a warp per rank). Only jump targets get a record, at their number j:
// run[j] = {target, its run's first node}, nx[j] = the number of the target that node's parent is
// (-1: none).
__global__ void __launch_bounds__(256) crit_runs_kernel(DevGraph g, const int32_t *__restrict__ parent,
                                                        const uint32_t *__restrict__ tgt,
                                                        const int32_t *__restrict__ wpre, int2 *__restrict__ run,
                                                        int32_t *__restrict__ nx) {
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
      if (i < re && ((tgt[i >> 5] >> (i & 31)) & 1u)) {
        const int32_t q = parent[x], j = crit_tidx(tgt, wpre, i);
        run[j] = make_int2(i, x);
        nx[j] = q < 0 ? -1 : crit_tidx(tgt, wpre, q);
      }
      carry = __shfl_sync(0xffffffffu, x, 31);
    }
  }
}

// step 6: the walk from the lowest node finishing at T is the list of runs j0 -> nx[j0] -> ...
// Followed one hop at a time it is one dependent L2 load per run (most path nodes are runs of
// their own: ~3k hops, ~0.45 ms for C5), so the list is ranked by pointer doubling instead:
// level l holds nx^(2^l); level l is built only while the list from j0 is longer than 2^(l-1)
// hops (level l-1 at j0 is not the end), so ~log2(path runs) passes of one thread per target.
// j0p[0] = the start node's number, j0p[1] = the number of targets (records 0 .. j0p[1] - 1 exist)
__global__ void __launch_bounds__(256) crit_j0_kernel(const int32_t *__restrict__ start_node, int32_t N,
                                                      const uint32_t *__restrict__ tgt, const int32_t *__restrict__ wpre,
                                                      int64_t nw, int32_t *__restrict__ j0) {
  const int32_t s = *start_node;
  j0[0] = (s < 0 || s >= N) ? -1 : crit_tidx(tgt, wpre, s);  // empty graph: empty path
  j0[1] = wpre[nw - 1] + __popc(tgt[nw - 1]);
  j0[2] = 0;  // set once a level finds the list covered; later levels are then not built
}
__global__ void __launch_bounds__(256) crit_double_kernel(int32_t l, int64_t T, int32_t *j0p,
                                                          int32_t *__restrict__ nx) {
  const int32_t j0 = j0p[0], cnt = j0p[1];
  const int32_t *prev = nx + (int64_t)(l - 1) * T;
  if (__ldcg(j0p + 2)) return;  // an earlier level covered the list; level l - 1 was not built
  if (j0 < 0 || __ldcg(prev + j0) < 0) {  // levels < l cover the list
    if (threadIdx.x == 0) j0p[2] = 1;
    return;
  }
  int32_t *cur = nx + (int64_t)l * T;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cnt; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = __ldcg(prev + j);
    cur[j] = a < 0 ? -1 : __ldcg(prev + a);
  }
}
// One CTA: the list's length H (greedy descent through the levels), then positions p = 0..H-1 in
// chunks of blockDim: run p = nx^p(j0) by p's binary digits, its node count, a block scan of the
// counts, and the run written out last node first.
__global__ void __launch_bounds__(1024) crit_emit_kernel(const int32_t *__restrict__ j0p, int64_t T, int32_t L,
                                                         const int32_t *__restrict__ nx, const int2 *__restrict__ run,
                                                         int32_t *__restrict__ path, int64_t cap,
                                                         int64_t *__restrict__ len_out) {
  __shared__ int32_t s_lu, s_h;
  __shared__ int64_t warp_sum[32];
  __shared__ int64_t s_carry;
  const int32_t j0 = *j0p;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    int32_t lu = 0, h = 0;
    if (j0 >= 0) {
      lu = 1;  // levels [0, lu) are built and cover the list
      while (lu < L && __ldcg(nx + (int64_t)(lu - 1) * T + j0) >= 0) ++lu;
      int32_t cur = j0;
      for (int32_t r = lu - 1; r >= 0; --r) {
        const int32_t nxt = __ldcg(nx + (int64_t)r * T + cur);
        if (nxt >= 0) {
          cur = nxt;
          h += 1 << r;
        }
      }
      h += 1;
    }
    s_lu = lu;
    s_h = h;
    s_carry = 0;
  }
  __syncthreads();
  const int32_t lu = s_lu, H = s_h;
  for (int32_t base = 0; base < H; base += blockDim.x) {
    const int32_t p = base + tid;
    int2 e = make_int2(0, 1);  // empty run
    if (p < H) {
      int32_t cur = j0;
      for (int32_t r = 0; r < lu; ++r)
        if ((p >> r) & 1) cur = __ldcg(nx + (int64_t)r * T + cur);
      e = __ldcg(run + cur);
    }
    const int64_t cnt = (int64_t)e.x - e.y + 1;
    int64_t inc = cnt;
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t v = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += v;
    }
    if (lane == 31) warp_sum[wid] = inc;
    __syncthreads();
    int64_t off0 = s_carry + inc - cnt;
    for (int i = 0; i < wid; ++i) off0 += warp_sum[i];
    for (int64_t i = 0; i < cnt; ++i)
      if (off0 + i < cap) path[off0 + i] = e.x - (int32_t)i;
    __syncthreads();
    if (tid == 0) {
      int64_t t = 0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += warp_sum[i];
      s_carry += t;
    }
    __syncthreads();
  }
  if (tid == 0) *len_out = s_carry;
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

static int64_t crit_targets(const DevGraph &g) { return g.G + 1 + (g.ms ? g.N : 0); }
static int32_t crit_levels(int64_t T) {  // levels of nx^(2^l) that rank any list over T targets
  int32_t L = 1;
  while (L < 31 && (1LL << L) < T + 1) ++L;
  return L;
}

size_t crit_scratch_bytes(const DevGraph &g, int64_t path_cap) {
  const int64_t nw = g.N / 32 + 1, nb = (nw + kScanWords - 1) / kScanWords, T = crit_targets(g);
  return 64 + (size_t)g.G * 12 + (size_t)g.N * 4 + (size_t)(2 * nw + nb) * 4 + 16 + (size_t)T * 8 +
         (size_t)T * crit_levels(T) * 4 + (size_t)std::max<int64_t>(path_cap, 1) * 4 + 64;
}

cudaError_t launch_critical_path(const DevGraph &g, const ScenParams &p, const int64_t *fin, int32_t Sp, int32_t k,
                                 int64_t *iter, bool have_T, void *scratch, int32_t *path_len_start[3],
                                 int64_t cap, cudaStream_t st) {
  // scratch: [start node][pad][j0, target count, done][pad][len][gkey G][gbest G][parent N][tgt nw][wpre nw][bsum nb][run T][nx L x T][path]
  const int64_t nw = g.N / 32 + 1, nb = (nw + kScanWords - 1) / kScanWords, T = crit_targets(g);
  const int32_t L = crit_levels(T);
  char *b = (char *)scratch;
  int32_t *start = (int32_t *)b;
  int32_t *j0 = start + 2;
  int64_t *len_out = (int64_t *)(b + 24);
  int64_t *gkey = (int64_t *)(b + 64);
  int32_t *gbest = (int32_t *)(gkey + g.G);
  int32_t *parent = gbest + g.G;
  uint32_t *tgt = (uint32_t *)(parent + g.N);
  int32_t *wpre = (int32_t *)(tgt + nw);
  int32_t *bsum = wpre + nw;
  int2 *run = (int2 *)(((uintptr_t)(bsum + nb) + 15) & ~(uintptr_t)15);
  int32_t *nx = (int32_t *)(run + T);
  int32_t *path = nx + (int64_t)L * T;
  path_len_start[0] = path;
  path_len_start[1] = (int32_t *)len_out;
  path_len_start[2] = start;
  cudaError_t e = cudaMemsetAsync(start, 0x7F, 4, st);
  if (e == cudaSuccess && !have_T) e = cudaMemsetAsync(iter + k, 0, 8, st);
  if (e == cudaSuccess && g.G > 0) e = cudaMemsetAsync(gkey, 0, (size_t)g.G * 8, st);
  if (e == cudaSuccess && g.G > 0) e = cudaMemsetAsync(gbest, 0x7F, (size_t)g.G * 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(tgt, 0, (size_t)nw * 4, st);
  if (e != cudaSuccess) return e;
  const int blocks = num_sms() * 8;
  if (g.N > 0 && !have_T) view_max_kernel<<<blocks, 256, 0, st>>>(g, fin, Sp, k, iter + k);
  if (g.N > 0) crit_start_kernel<<<blocks, 256, 0, st>>>(g, fin, Sp, k, iter, start);
  if (g.G > 0) {
    crit_ready_kernel<<<blocks, 256, 0, st>>>(g, fin, Sp, k, iter, gkey);
    crit_tie_kernel<<<blocks, 256, 0, st>>>(g, fin, Sp, k, iter, gkey, gbest);
    crit_gfin_kernel<<<blocks, 256, 0, st>>>(g, p, fin, Sp, k, iter, gkey, gbest, tgt);
  }
  if (g.N > 0) crit_parent_kernel<<<blocks, 256, 0, st>>>(g, fin, Sp, k, gkey, gbest, parent, start, tgt);
  crit_bsum_kernel<<<(unsigned)nb, 256, 0, st>>>(tgt, nw, bsum);
  crit_wpre_kernel<<<(unsigned)nb, 256, 0, st>>>(tgt, nw, bsum, wpre);
  if (g.W > 0) crit_runs_kernel<<<blocks, 256, 0, st>>>(g, parent, tgt, wpre, run, nx);
  crit_j0_kernel<<<1, 1, 0, st>>>(start, (int32_t)g.N, tgt, wpre, nw, j0);
  const int dblocks = (int)std::min<int64_t>(blocks, (T + 255) / 256);
  for (int32_t l = 1; l < L; ++l) crit_double_kernel<<<dblocks, 256, 0, st>>>(l, T, j0, nx);
  crit_emit_kernel<<<1, 1024, 0, st>>>(j0, T, L, nx, run, path, cap, len_out);
  return cudaGetLastError();
}

}  // namespace prism
