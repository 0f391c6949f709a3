// expand.cu — rows a1-a4: rank coordinates, template expansion into the node SoA, and the
// sync-group CSR (collective instances + P2P messages -> member node ids).
//
// Every store here is a coalesced streaming write of the CSR DAG; the per-stage template tables
// (a few hundred KB) stay L2-resident and are read by every rank of their stage ("execution
// graphs are identical across DP groups" -> the expander copies one template per stage into every
// rank's node range). Algorithmic bytes: 41 B per node + 8 B per membership + 24 B per group
// (DESIGN.md §6).
#include <cuda_runtime.h>

#include <algorithm>

#include "graph.h"

namespace prism {

namespace {

// Row a1: rank -> (tp, pp, dp) under the rank order (reading Z1); ep/edp carved from dp.
__device__ __forceinline__ int32_t stage_of(const DevGraph &g, int32_t r) {
  return g.order == PRISM_ORDER_MEGATRON ? r / (g.tp * g.dp) : (r / g.tp) % g.pp;
}
__device__ __forceinline__ int32_t rank_of(const DevGraph &g, int32_t tp_i, int32_t pp_i, int32_t dp_i) {
  return g.order == PRISM_ORDER_MEGATRON ? tp_i + g.tp * (dp_i + g.dp * pp_i)
                                         : tp_i + g.tp * (pp_i + g.pp * dp_i);
}

// Exclusive scans of per-rank node / slot counts (one block of 1024 threads, 1024 ranks per
// round: warp shuffle scans, then a scan of the 32 warp totals; W <= 2^30 but small in practice).
__global__ void __launch_bounds__(1024) rank_tables_kernel(DevGraph g) {
  __shared__ int64_t w_nodes[32], w_slots[32];
  __shared__ int64_t carry_n, carry_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_n = carry_s = 0;
  __syncthreads();
  for (int32_t base = 0; base < g.W; base += 1024) {
    const int32_t r = base + threadIdx.x;
    int64_t n = 0, sl = 0;
    if (r < g.W) {
      const int32_t s = stage_of(g, r);
      g.rank_stage[r] = s;
      n = g.t_len[s];
      sl = g.t_slots_total[s];
    }
    int64_t xn = n, xs = sl;  // inclusive scans within the warp
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t yn = __shfl_up_sync(0xffffffffu, xn, off), ys = __shfl_up_sync(0xffffffffu, xs, off);
      if (lane >= off) {
        xn += yn;
        xs += ys;
      }
    }
    if (lane == 31) {
      w_nodes[wid] = xn;
      w_slots[wid] = xs;
    }
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the warp totals
      int64_t tn = w_nodes[lane], ts = w_slots[lane];
      int64_t un = tn, us = ts;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int64_t yn = __shfl_up_sync(0xffffffffu, un, off), ys = __shfl_up_sync(0xffffffffu, us, off);
        if (lane >= off) {
          un += yn;
          us += ys;
        }
      }
      w_nodes[lane] = un - tn;
      w_slots[lane] = us - ts;
    }
    __syncthreads();
    if (r < g.W) {
      g.rank_ptr[r] = (int32_t)(carry_n + w_nodes[wid] + xn - n);
      g.rank_slot[r] = (int32_t)(carry_s + w_slots[wid] + xs - sl);
    }
    __syncthreads();
    if (threadIdx.x == 1023) {  // the round's totals
      carry_n += w_nodes[31] + xn;
      carry_s += w_slots[31] + xs;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    g.rank_ptr[g.W] = (int32_t)carry_n;
    g.rank_slot[g.W] = (int32_t)carry_s;
    g.node_gptr[g.N] = (int32_t)carry_s;
    g.grp_ptr[g.G] = (int32_t)g.M;
  }
}

// Concrete group id (uid field) of instance `inst` of quotient group q (closed form, a2).
__device__ __forceinline__ uint64_t group_gid(const DevGraph &g, const QGroup &q, int32_t inst) {
  const int32_t s = q.stage;
  switch (q.type) {
    case PRISM_ROLE_TP: return (uint64_t)s + (uint64_t)g.pp * inst;                    // inst = dp
    case PRISM_ROLE_DP: return (uint64_t)inst + (uint64_t)g.tp * s;                    // inst = tp
    case PRISM_ROLE_EP:                                                                  // (tp, edp)
      return (uint64_t)(inst % g.tp) + (uint64_t)g.tp * (s + (uint64_t)g.pp * (inst / g.tp));
    case PRISM_ROLE_EDP:                                                                 // (tp, ep)
      return (uint64_t)(inst % g.tp) + (uint64_t)g.tp * (s + (uint64_t)g.pp * (inst / g.tp));
    case PRISM_ROLE_WORLD: return 0;
    default: {  // P2P message: sender rank * 2 + direction
      const int32_t sender = rank_of(g, inst % g.tp, s, inst / g.tp);
      return (uint64_t)sender * 2 + q.dir;
    }
  }
}
__device__ __forceinline__ uint64_t group_uid(const DevGraph &g, const QGroup &q, int32_t inst) {
  return ((uint64_t)q.type << 56) | (group_gid(g, q, inst) << 24) | (uint64_t)q.occ;
}

// Row e: the shards holding a member of the group of a rank with DP coordinates (dpi, epi, edpi)
// under the DP-block sharding (shard of dp_i = dp_i / (dp / n_shards)); TP groups and P2P
// messages stay inside one DP coordinate, hence inside one shard. Under PP-stage blocks (shard of
// pp_i = pp_i / (pp / n_shards)) every collective but WORLD stays inside its stage; a P2P message
// joins the sender's and the receiver's stage blocks.
__device__ __forceinline__ uint32_t shard_mask(const DevGraph &g, const QGroup &q, int32_t dpi, int32_t epi,
                                               int32_t edpi) {
  const int32_t type = q.type;
  if (g.shard_axis == 1) {
    const int32_t Bp = g.pp / g.n_shards;
    if (type == PRISM_ROLE_WORLD) return g.n_shards >= 32 ? 0xFFFFFFFFu : (1u << g.n_shards) - 1u;
    if (type == PRISM_ROLE_P2P) return (1u << (q.stage / Bp)) | (1u << (q.stage2 / Bp));
    return 1u << (q.stage / Bp);
  }
  const int32_t B = g.dp / g.n_shards;
  switch (type) {
    case PRISM_ROLE_DP:
    case PRISM_ROLE_WORLD: return g.n_shards >= 32 ? 0xFFFFFFFFu : (1u << g.n_shards) - 1u;
    case PRISM_ROLE_EP: {  // members dp = edpi*ep + j, j < ep: a contiguous block
      const int32_t a = (edpi * g.ep) / B, b = (edpi * g.ep + g.ep - 1) / B;
      uint32_t m = 0;
      for (int32_t x = a; x <= b; ++x) m |= 1u << x;
      return m;
    }
    case PRISM_ROLE_EDP: {  // members dp = j*ep + epi, j < dp/ep
      uint32_t m = 0;
      for (int32_t j = 0; j < g.dp / g.ep; ++j) m |= 1u << ((j * g.ep + epi) / B);
      return m;
    }
    default: return 1u << (dpi / B);
  }
}

// Rows a3 + a4 (node side): one block per rank (grid-stride), threads over the rank's template
// ops, then over its template slots; every write is a coalesced run along the rank's nodes /
// membership slots. A slot's group instance and member index follow in closed form from the
// rank's coordinates (the same enumeration as the group side below).
// A quotient group through the read-only path (16-byte loads): the expansion's loads can then be
// scheduled ahead of its stores (plain loads would be ordered behind them, as they may alias).
__device__ __forceinline__ QGroup ldg_q(const QGroup *p) {
  static_assert(sizeof(QGroup) % 16 == 0, "QGroup is loaded as int4 words");
  QGroup q;
  const int4 *src = reinterpret_cast<const int4 *>(p);
  int4 *dst = reinterpret_cast<int4 *>(&q);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(QGroup) / 16); ++i) dst[i] = __ldg(src + i);
  return q;
}


// Template fields of one op that the node-side expansion writes (expand_nodes_kernel): the
// structure only (previous sync op, slot offset, stream / event edges); the op's own fields stay
// in the template tables (graph.h nd_*).
struct OpF {
  int32_t tps, tsp, sp, es;
  uint16_t msv;
};
__device__ __forceinline__ OpF load_opf(const DevGraph &g, int64_t ti) {
  OpF f;
  f.tps = __ldg(g.t_prev_sync + ti);
  f.tsp = __ldg(g.t_slot_ptr + ti);
  f.sp = -1;
  f.es = -1;
  f.msv = 0;
  if (g.ms) {  // row f2
    f.sp = g.t_spred[ti];
    f.es = g.t_esrc[ti];
    f.msv = g.t_ms[ti];
  }
  return f;
}

// One block per batch of kRanksPerBlock ranks of one stage: a thread loads template op i's fields
// (and its quotient group) once and writes node i of every rank of the batch, so the L2-resident
// template tables are read W / pp / kRanksPerBlock times instead of once per rank (the per-rank
// version moved 2.3 GB of template reads through L2 for 1.3 GB of graph writes on C5).
constexpr int kRanksPerBlock = 8;

__global__ void __launch_bounds__(256, 4) expand_nodes_kernel(DevGraph g) {
  __shared__ int32_t s_r[kRanksPerBlock], s_rb[kRanksPerBlock], s_slot0[kRanksPerBlock];
  __shared__ int32_t s_tpi[kRanksPerBlock], s_dpi[kRanksPerBlock];
  const int32_t per_stage = g.W / g.pp;  // tp * dp ranks run each stage template
  const int32_t nb = (per_stage + kRanksPerBlock - 1) / kRanksPerBlock;
  for (int32_t blk = blockIdx.x; blk < g.pp * nb; blk += gridDim.x) {
    const int32_t s = blk / nb, k0 = (blk - s * nb) * kRanksPerBlock;
    const int32_t nr = min(kRanksPerBlock, per_stage - k0);
    __syncthreads();  // the previous batch's readers are done with the shared rank table
    if (threadIdx.x < nr) {
      const int32_t kk = k0 + threadIdx.x;
      const int32_t tpi = kk % g.tp, dpi = kk / g.tp;
      const int32_t r = rank_of(g, tpi, s, dpi);
      s_r[threadIdx.x] = r;
      s_rb[threadIdx.x] = g.rank_ptr[r];
      s_slot0[threadIdx.x] = g.rank_slot[r];
      s_tpi[threadIdx.x] = tpi;
      s_dpi[threadIdx.x] = dpi;
    }
    __syncthreads();
    const int64_t op0 = g.t_op0[s];
    const int32_t len = (int32_t)g.t_len[s];
    // node side: template fields read once (coalesced SoA loads), written for every rank of the
    // batch (coalesced along each rank's nodes); the next op's fields are loaded before this op's
    // stores (software pipelined: the loads' latency overlaps the stores)
    OpF cur;
    if ((int32_t)threadIdx.x < len) cur = load_opf(g, op0 + threadIdx.x);
    for (int32_t i = threadIdx.x; i < len; i += blockDim.x) {
      OpF nxt;
      if (i + (int32_t)blockDim.x < len) nxt = load_opf(g, op0 + i + blockDim.x);
      for (int32_t j = 0; j < nr; ++j) {
        const int32_t r = s_r[j], rb = s_rb[j];
        const int32_t n = rb + i;
        // the op's own fields (duration, kind, label, memory, replay record) are the template's:
        // looked up by (stage, index) where needed (graph.h nd_*), not written per node
        g.node_rank[n] = r;
        g.node_prev_sync[n] = cur.tps < 0 ? -1 : rb + cur.tps;
        g.node_gptr[n] = s_slot0[j] + cur.tsp;
        if (g.ms) {
          g.node_ms[n] = cur.msv;
          g.node_spred[n] = cur.sp < 0 ? -1 : rb + cur.sp;
          g.node_esrc[n] = cur.es < 0 ? -1 : rb + cur.es;
        }
      }
      cur = nxt;
    }
    // slot side: one quotient group load per template slot, written for every rank of the batch
    const int64_t u0 = g.stage_slot0[s];
    const int32_t nsl = (int32_t)(g.stage_slot0[s + 1] - u0);
    for (int32_t u = threadIdx.x; u < nsl; u += blockDim.x) {
      const QGroup q = ldg_q(g.q + __ldg(g.slot_q + u0 + u));
      const int32_t role = __ldg(g.slot_role + u0 + u);
      const bool large = q.xbase < 0 && q.lbase >= 0;
      for (int32_t jr = 0; jr < nr; ++jr) {
        const int32_t tpi = s_tpi[jr], dpi = s_dpi[jr], epi = dpi % g.ep, edpi = dpi / g.ep;
        const int32_t inst = group_inst(g, q.type, tpi, dpi, epi, edpi);
        int32_t j;
        switch (q.type) {
          case PRISM_ROLE_TP: j = tpi; break;
          case PRISM_ROLE_DP: j = dpi; break;
          case PRISM_ROLE_EP: j = epi; break;
          case PRISM_ROLE_EDP: j = edpi; break;
          case PRISM_ROLE_WORLD: j = s_r[jr]; break;
          default: j = role; break;
        }
        const int32_t h = s_slot0[jr] + u;
        const int64_t grp = q.gbase + inst;
        g.node_grp[h] = (int32_t)grp;
        g.node_mslot[h] = (int32_t)(q.mbase + (int64_t)inst * q.size + j);
        g.h_base[h] = large ? (int32_t)(q.lbase + inst) : (q.xbase < 0 ? -1 : (int32_t)(q.xbase + (int64_t)inst * q.size));
        g.h_meta[h] = (uint32_t)min(q.size, 0xFFFF) | ((uint32_t)min(j, 0x7FFF) << 16) | (large ? 0x80000000u : 0u);
        g.h_dur[h] = q.dur;
        g.h_uid[h] = group_uid(g, q, inst);
        if (g.h_smask) g.h_smask[h] = shard_mask(g, q, dpi, epi, edpi);
      }
    }
  }
}

// Row a4 (group side): one block per chunk of 2048 memberships of one quotient group (host-made
// chunk table, no search); member node ids by closed form from the coordinates; coalesced writes
// of grp_mem and of the per-group arrays.
__global__ void __launch_bounds__(256) build_groups_kernel(DevGraph g) {
  for (int32_t c = blockIdx.x; c < g.nchunk; c += gridDim.x) {
    const QGroup &q = g.q[g.chunk_q[c]];
    const int64_t mq = (int64_t)q.inst * q.size;
    const int64_t m_end = min(mq, g.chunk_m[c] + 2048);
    const int32_t s = q.stage;
    for (int64_t local = g.chunk_m[c] + threadIdx.x; local < m_end; local += blockDim.x) {
      // local < M < 2^31 (checked by the plan): 32-bit division
      const int32_t inst = (int32_t)local / q.size;
      const int32_t j = (int32_t)local - inst * q.size;
      const int64_t m = q.mbase + local;
      const int64_t grp = q.gbase + inst;
      int32_t rank, tidx = q.tidx;
      switch (q.type) {
        case PRISM_ROLE_TP: rank = rank_of(g, j, s, inst); break;
        case PRISM_ROLE_DP: rank = rank_of(g, inst, s, j); break;
        case PRISM_ROLE_EP: rank = rank_of(g, inst % g.tp, s, (inst / g.tp) * g.ep + j); break;
        case PRISM_ROLE_EDP: rank = rank_of(g, inst % g.tp, s, j * g.ep + inst / g.tp); break;
        case PRISM_ROLE_WORLD:
          rank = j;
          tidx = g.wpos[q.wpos + g.rank_stage[j]];
          break;
        default:  // P2P message: member 0 = sender, member 1 = receiver (same tp/dp coords)
          if (j == 0) {
            rank = rank_of(g, inst % g.tp, s, inst / g.tp);
          } else {
            rank = rank_of(g, inst % g.tp, q.stage2, inst / g.tp);
            tidx = q.tidx2;
          }
          break;
      }
      g.grp_mem[m] = g.rank_ptr[rank] + tidx;
      if (j == 0) {
        g.grp_ptr[grp] = (int32_t)m;
        g.grp_dur[grp] = q.dur;
        g.grp_level[grp] = q.level;
        g.grp_uid[grp] = group_uid(g, q, inst);
        g.grp_xbase[grp] = q.xbase < 0 ? -1 : q.xbase + (int64_t)inst * q.size;
        g.grp_lidx[grp] = q.lbase < 0 ? -1 : (int32_t)(q.lbase + inst);
      }
    }
  }
}

}  // namespace

// Replica cells: one thread per (stage, DP block, cross op of the stage); cell-full ops get their
// group's cell-level slot (row a4 at cell granularity). The cell's member index in its group: DP
// and EDP (ep = 1) groups number their cells by DP block, EP groups by the block within the EP
// group, the WORLD group by (stage, block).
__global__ void __launch_bounds__(256) cell_records_kernel(DevGraph g) {
  const int32_t R = g.cell_R, nb = g.dp / R;
  for (int32_t s = blockIdx.x; s < g.pp; s += gridDim.x) {
    const int32_t x0 = g.x_ptr[s], nx = g.x_ptr[s + 1] - x0;
    for (int32_t y = threadIdx.x; y < nb * nx; y += blockDim.x) {
      const int32_t b = y / nx, x = x0 + y % nx;
      const XOp xo = g.x_ops[x];
      if (!(xo.flags & 1)) continue;
      const QGroup q = ldg_q(g.q + __ldg(g.t_q0 + g.t_op0[s] + xo.tidx));
      const int32_t dpi = b * R, epi = dpi % g.ep, edpi = dpi / g.ep;
      const int32_t inst = group_inst(g, q.type, 0, dpi, epi, edpi);
      const int32_t cz = q.size / R;
      int32_t own;
      switch (q.type) {
        case PRISM_ROLE_EP: own = epi / R; break;
        case PRISM_ROLE_WORLD: own = s * nb + b; break;
        default: own = b; break;  // DP, EDP with ep = 1
      }
      const bool large = q.clbase >= 0;
      const int64_t rec = g.crec_ptr[s] + (int64_t)b * nx + (x - x0);
      g.c_meta[rec] = (uint32_t)min(cz, 0xFFFF) | ((uint32_t)min(own, 0x7FFF) << 16) | (large ? 0x80000000u : 0u);
      g.c_base[rec] = large ? (int32_t)(q.clbase + inst) : (int32_t)(q.cxbase + (int64_t)inst * cz);
    }
  }
}

// Test hook (prism_debug_export): the per-node template fields, materialised.
__global__ void __launch_bounds__(256) materialize_kernel(DevGraph g, int32_t which, void *out) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < g.N; n += (int64_t)gridDim.x * blockDim.x) {
    const int32_t m = (int32_t)n;
    switch (which) {
      case 2: ((int64_t *)out)[n] = nd_dur(g, m); break;
      case 3: ((uint8_t *)out)[n] = nd_kind(g, m); break;
      case 4: ((uint32_t *)out)[n] = nd_label(g, m); break;
      case 5: ((int64_t *)out)[n] = nd_alloc(g, m); break;
      default: ((int64_t *)out)[n] = nd_free(g, m); break;
    }
  }
}

cudaError_t launch_materialize(const DevGraph &g, int32_t which, void *out, cudaStream_t st) {
  if (g.N > 0) materialize_kernel<<<num_sms() * 4, 256, 0, st>>>(g, which, out);
  return cudaGetLastError();
}

cudaError_t launch_cell_records(const DevGraph &g, cudaStream_t st) {
  if (g.cell_R > 1 && g.pp > 0) cell_records_kernel<<<g.pp, 256, 0, st>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_expand(const DevGraph &g, cudaStream_t st) {
  rank_tables_kernel<<<1, 1024, 0, st>>>(g);
  if (g.N > 0) {
    const int64_t batches = (int64_t)g.pp * ((g.W / g.pp + kRanksPerBlock - 1) / kRanksPerBlock);
    const int blocks = (int)std::min<int64_t>(batches, num_sms() * 16);
    expand_nodes_kernel<<<blocks, 256, 0, st>>>(g);
  }
  if (g.M > 0 && g.nchunk > 0) build_groups_kernel<<<g.nchunk, 256, 0, st>>>(g);
  return cudaGetLastError();
}

}  // namespace prism
