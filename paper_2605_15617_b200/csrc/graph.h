// graph.h — the device-resident graph (row a3/a4 output) and launch wrappers of every kernel.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "prism_internal.h"

namespace prism {

// Plain device pointers; passed by value to kernels.
struct DevGraph {
  int32_t W, pp, tp, dp, ep, order;
  // row e: this shard replays the ranks with dp_i in [d0, d1) and pp_i in [s0, s1) (everything
  // unsharded); shard_axis 0 = DP blocks (d0/d1 vary), 1 = PP-stage blocks (s0/s1 vary)
  int32_t n_shards, shard, d0, d1, s0, s1, shard_axis;
  // rows f1/f3/f4: node_sdur / h_dur / node_dur / grp_dur point at per-node override arrays and
  // compute spans / chained collectives last their own rank's value (prism_set_durations)
  int32_t per_rank_dur;
  // device watchdog of the waiting replay kernels (prism_debug_set): abort with PRISM_E_DEADLOCK
  // after watchdog_ns without progress; stall_unit >= 0 makes that warp of the next replays
  // return at once (test hook: forces the watchdog)
  int32_t stall_unit;
  uint64_t watchdog_ns;
  // fin rows kept by this graph: [fin_node0, fin_node0 + fin_rows) of the row order below
  int64_t fin_node0, fin_rows;
  // replica cells (cell_R > 1, tp = 1): a cell is cell_R consecutive DP replicas of one stage;
  // crec_ptr[s] + b * (x ops of stage s) + x = the cell record of cross op x of cell (s, b):
  // c_meta = size in cells | own cell index << 16 | large << 31, c_base = first cell-level ready
  // slot or the accumulator index of the op's group (cell-full ops, XOp flags bit 0)
  int32_t cell_R;
  int32_t cta_ks;            // EP CTAs: the cta_ks replica cells of one EP group share a CTA
  int64_t Ltot;              // ops of all stage templates together
  const int64_t *crec_ptr;   // [pp+1]
  int32_t *c_base;
  uint32_t *c_meta;
  // row f2: multi-stream ranks (per-node stream / event fields, directional predecessors, -1 =
  // none); streams and densely renumbered event slots used by the graph
  int32_t ms, ms_streams, ms_events;
  const uint16_t *t_ms;      // per template op: stream | ev_record << 4 | ev_wait << 8
  const int32_t *t_spred;    // per template op: previous op of its stream (template index)
  const int32_t *t_esrc;     // per template op: event source (template index)
  uint16_t *node_ms;         // [N] (multi-stream graphs only)
  int32_t *node_spred;       // [N]
  int32_t *node_esrc;        // [N]
  int64_t N, G, M;
  // rank tables
  int32_t *rank_ptr;        // [W+1] first node of each rank
  int32_t *rank_slot;       // [W+1] first membership slot (node_grp) of each rank
  int32_t *rank_stage;      // [W]
  // node SoA
  int32_t *node_rank;       // [N]
  int64_t *node_dur;        // [N]
  uint8_t *node_kind;       // [N]
  uint32_t *node_label;     // [N]
  int64_t *node_alloc;      // [N]
  int64_t *node_free;       // [N]
  int32_t *node_prev_sync;  // [N]
  int32_t *node_gptr;       // [N+1]
  int32_t *node_grp;        // [M]
  // sync-group CSR (sorted by level)
  int32_t *grp_ptr;         // [G+1]
  int32_t *grp_mem;         // [M]
  int64_t *grp_dur;         // [G]
  uint64_t *grp_uid;        // [G]
  int32_t *grp_level;       // [G]
  // replay v2 (cell kernel) support
  int32_t *node_mslot;      // [M] membership index of each node slot (parallel to node_grp)
  // per-node replay record (written by the expander): what the chain walk needs, coalesced
  uint8_t *node_cls;        // [N] 0 compute span, 1 in-cell (TP) collective, 2 cross-cell sync
  int64_t *node_sdur;       // [N] compute: own duration; single-group sync: the group's duration
  uint64_t *node_uid;       // [N] perturbation uid: (rank<<32)|tidx, or the (first) group's uid
  int64_t *grp_xbase;       // [G] first ready slot (small cross-cell group), else -1
  int32_t *grp_lidx;        // [G] accumulator index (large cross-cell group), else -1
  // per membership slot h (parallel to node_grp): flat sync record for the cell kernel
  int32_t *h_base;          // small group: first ready slot of the group; large: accumulator index
  uint32_t *h_meta;         // size (bits 0-15) | own member offset (16-30) | large (bit 31)
  int64_t *h_dur;           // the group's duration
  uint64_t *h_uid;          // the group's perturbation uid
  uint32_t *h_smask;        // sharded graphs: bit m = shard m holds a member of the slot's group
  int64_t M_cross, G_large;
  // per-stage template tables (tiny; L2 resident)
  int64_t *t_op0;           // [pp] first op of each stage
  int64_t *t_len;           // [pp]
  int32_t *t_prev_sync;     // per op
  int32_t *t_slot_ptr;      // per op
  int64_t *t_slots_total;   // [pp]
  int64_t *static_mem;      // [pp]
  const QGroup *q;          // quotient groups (level order)
  int32_t nq;
  // per template slot (stage-major, stage s at stage_slot0[s]) and group-side build chunks
  const int64_t *stage_slot0;
  const int32_t *slot_q;
  const int32_t *slot_tidx;
  const uint8_t *slot_role;
  const uint8_t *slot_first;
  const int32_t *chunk_q;
  const int64_t *chunk_m;
  int32_t nchunk;
  const int32_t *wpos;      // WORLD per-stage template indices
  const uint8_t *t_cls;     // replay class per template op (Plan::t_cls)
  const int32_t *t_q0;      // per template op: quotient group of its first slot (-1: compute)
  // per template op, structure-of-arrays copies of the prism_op fields the expansion writes, and
  // the replay-record duration (compute span: dur_ns; sync node: its first group's duration)
  const int64_t *t_dur, *t_alloc, *t_free, *t_sdur;
  const uint32_t *t_label;
  const uint8_t *t_kind;
  // per template op: its first quotient group's type | dir << 8 | stage << 16 | occurrence << 32
  // (0 for compute spans): what the node's replay uid needs, without the 96-byte QGroup
  const uint64_t *t_qinfo;
  const int32_t *x_ptr;     // [pp+1] cross-op list of each stage
  const XOp *x_ops;
};

// Layout of the recorded finish times fin. Rows are nodes in CELL-INTERLEAVED
// order: the tp ranks of a (stage, dp) cell run one template, so op i of the cell's rank tp_i is
// row cell_first_node + i * tp + tp_i (a cell's rows are one contiguous block either way, so a DP
// block's rows stay contiguous for sharding). Scenarios are grouped in chunks of cw = min(32, Sp)
// lanes, chunk-major: element (row, k) sits at ((k / cw) * rows + row - node0) * cw + k % cw. A
// cell kernel warp (one cell, one 32-scenario chunk) thus writes op i of its ranks as C
// consecutive 256-byte rows at constant offsets (no per-op address arithmetic), and its ops follow
// each other contiguously.
// Replica cells (cell_R = R > 1, tp = 1) interleave the R replicas instead: op i of replica rr of
// cell (stage s, DP block b) is row base(s, b) + i R + rr with base = R (b Ltot + op0[s]) under
// TP_PP_DP (cells b-major, then s) and dp op0[s] + b R len(s) under Megatron order.
#ifdef __CUDACC__
__device__ __forceinline__ int64_t cell_row0(const DevGraph &g, int32_t r) {  // row of rank r's op 0
  if (g.cell_R <= 1) {
    const int32_t tpi = r % g.tp;
    return (int64_t)g.rank_ptr[r - tpi] + tpi;
  }
  const int32_t R = g.cell_R;
  const bool meg = g.order == PRISM_ORDER_MEGATRON;
  const int32_t s = meg ? r / g.dp : r % g.pp, dpi = meg ? r % g.dp : r / g.pp;
  const int64_t base = meg ? (int64_t)g.dp * g.t_op0[s] + (int64_t)(dpi / R) * R * g.t_len[s]
                           : (int64_t)R * ((int64_t)(dpi / R) * g.Ltot + g.t_op0[s]);
  return base + dpi % R;
}
__device__ __forceinline__ int32_t cell_row_stride(const DevGraph &g) { return g.cell_R > 1 ? g.cell_R : g.tp; }
__device__ __forceinline__ int64_t fin_row(const DevGraph &g, int32_t n) {
  const int32_t r = g.node_rank[n];
  return cell_row0(g, r) + (int64_t)(n - g.rank_ptr[r]) * cell_row_stride(g);
}
__device__ __forceinline__ int64_t fin_off(const DevGraph &g, int64_t row, int32_t k, int32_t Sp) {
  const int32_t cw = Sp < 32 ? Sp : 32;
  return ((int64_t)(k / cw) * g.fin_rows + (row - g.fin_node0)) * cw + (k % cw);
}
#endif

// ---- closed forms and template lookups shared by the kernels (rows a1-a4) ----------------------
#ifdef __CUDACC__
__device__ __forceinline__ int32_t dg_rank_of(const DevGraph &g, int32_t tp_i, int32_t pp_i, int32_t dp_i) {
  return g.order == PRISM_ORDER_MEGATRON ? tp_i + g.tp * (dp_i + g.dp * pp_i) : tp_i + g.tp * (pp_i + g.pp * dp_i);
}
// Instance of quotient group q that a rank with these coordinates joins (closed form, a2).
__device__ __forceinline__ int32_t group_inst(const DevGraph &g, int32_t type, int32_t tpi, int32_t dpi,
                                              int32_t epi, int32_t edpi) {
  switch (type) {
    case PRISM_ROLE_TP: return dpi;
    case PRISM_ROLE_DP: return tpi;
    case PRISM_ROLE_EP: return tpi + g.tp * edpi;
    case PRISM_ROLE_EDP: return tpi + g.tp * epi;
    case PRISM_ROLE_WORLD: return 0;
    default: return tpi + g.tp * dpi;  // P2P message (sender or receiver: same tp/dp)
  }
}
// The same from a host-packed t_qinfo word (type | dir << 8 | stage << 16 | occurrence << 32).
__device__ __forceinline__ uint64_t group_uid_packed(const DevGraph &g, uint64_t qi, int32_t inst) {
  const int32_t type = (int32_t)(qi & 0xFF), dir = (int32_t)((qi >> 8) & 0xFF);
  const int32_t s = (int32_t)((qi >> 16) & 0xFFFF);
  uint64_t gid;
  switch (type) {
    case PRISM_ROLE_TP: gid = (uint64_t)s + (uint64_t)g.pp * inst; break;
    case PRISM_ROLE_DP: gid = (uint64_t)inst + (uint64_t)g.tp * s; break;
    case PRISM_ROLE_EP:
    case PRISM_ROLE_EDP: gid = (uint64_t)(inst % g.tp) + (uint64_t)g.tp * (s + (uint64_t)g.pp * (inst / g.tp)); break;
    case PRISM_ROLE_WORLD: gid = 0; break;
    default: gid = (uint64_t)dg_rank_of(g, inst % g.tp, s, inst / g.tp) * 2 + dir; break;
  }
  return ((uint64_t)type << 56) | (gid << 24) | (qi >> 32);
}

// Per-node fields that are the node's template op's (every rank of a stage runs the stage's
// template): looked up from the L2-resident per-stage tables instead of being written out
// per node by the expansion; an override array (prism_set_durations / _set_moe_load) takes their
// place when set.
__device__ __forceinline__ int64_t node_op(const DevGraph &g, int32_t n) {
  const int32_t r = g.node_rank[n];
  return g.t_op0[g.rank_stage[r]] + (n - g.rank_ptr[r]);
}
__device__ __forceinline__ int64_t nd_dur(const DevGraph &g, int32_t n) {
  return g.node_dur ? g.node_dur[n] : __ldg(g.t_dur + node_op(g, n));
}
__device__ __forceinline__ int64_t nd_alloc(const DevGraph &g, int32_t n) {
  return g.node_alloc ? g.node_alloc[n] : __ldg(g.t_alloc + node_op(g, n));
}
__device__ __forceinline__ int64_t nd_free(const DevGraph &g, int32_t n) {
  return g.node_free ? g.node_free[n] : __ldg(g.t_free + node_op(g, n));
}
__device__ __forceinline__ uint8_t nd_kind(const DevGraph &g, int32_t n) { return __ldg(g.t_kind + node_op(g, n)); }
__device__ __forceinline__ uint32_t nd_label(const DevGraph &g, int32_t n) { return __ldg(g.t_label + node_op(g, n)); }
#endif

// ---- TMA (cp.async.bulk) 1-D copies global -> shared, completed on an mbarrier ------------------
#ifdef __CUDACC__
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");  // visible to the async proxy
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
// bytes: a multiple of 16; src and dst 16-byte aligned
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
      ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}
#endif

// Scenario parameters as seen by the kernels.
struct ScenParams {
  int32_t S;         // scenarios
  int32_t first;     // global index of local scenario 0 (perturbation key k = first + local)
  int32_t amp;       // amp_q16
  uint64_t seed;
  uint32_t mask;     // kind mask
  int32_t record;    // write fin[N][S]
  int32_t mod;       // 2*amp+1
  uint64_t mod_magic;  // Lemire fastmod constant for mod (x < 2^32)
  uint32_t mod_m32;    // ceil(2^32 / mod): 32-bit quotient estimate for x < 2^24 (perturb_x)
  uint32_t pad;
};

// Reading Z8's perturbation with the splitmix64 hash x already mixed: v = splitmix64(x) >> 40
// (the finaliser's last xorshift leaves bits 40..63 unchanged, so it is skipped), r = v mod (2 amp
// + 1), d' = (d * (65536 + r - amp)) >> 16. The mod of the 24-bit v uses q = umulhi(v, ceil(2^32 /
// mod)): q overshoots floor(v / mod) by at most one (v * (M - 2^32/mod) / 2^32 < 2^-8), so one
// conditional add of mod makes r exact.
#ifdef __CUDACC__
__device__ __forceinline__ int64_t perturb_x(int64_t d, uint64_t x, const ScenParams &p) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  const uint32_t v = (uint32_t)(z >> 40);
  int32_t r = (int32_t)(v - __umulhi(v, p.mod_m32) * (uint32_t)p.mod);
  if (r < 0) r += p.mod;
  return (d * (int64_t)((uint32_t)r + (uint32_t)(65536 - p.amp))) >> 16;
}

// The same function for C independent (d, x) pairs, t[r] += perturb_x(d[r], x[r]), written step by
// step across r (structure of arrays): ptxas otherwise emits the C hash chains one after another,
// and a lone warp pays each chain's full dependency latency (958 vs 603 cycles per 8-rank op,
// tools/micro/hashop.cu). The top word of the last product is formed from 32-bit halves:
// hi32(y * M) = umulhi(lo, M_lo) + lo * M_hi + hi * M_lo (mod 2^32).
template <int C>
__device__ __forceinline__ void perturb_add(int64_t (&t)[C], const int64_t (&d)[C], const uint64_t (&x)[C],
                                            const ScenParams &p) {
  uint64_t z[C];
#pragma unroll
  for (int r = 0; r < C; ++r) z[r] = x[r] + 0x9E3779B97F4A7C15ULL;
#pragma unroll
  for (int r = 0; r < C; ++r) z[r] = (z[r] ^ (z[r] >> 30)) * 0xBF58476D1CE4E5B9ULL;
#pragma unroll
  for (int r = 0; r < C; ++r) z[r] = z[r] ^ (z[r] >> 27);
  uint32_t v[C];
#pragma unroll
  for (int r = 0; r < C; ++r) {
    const uint32_t lo = (uint32_t)z[r], hi = (uint32_t)(z[r] >> 32);
    v[r] = (__umulhi(lo, 0x133111EBu) + lo * 0x94D049BBu + hi * 0x133111EBu) >> 8;
  }
  int32_t m[C];
#pragma unroll
  for (int r = 0; r < C; ++r) m[r] = (int32_t)(v[r] - __umulhi(v[r], p.mod_m32) * (uint32_t)p.mod);
#pragma unroll
  for (int r = 0; r < C; ++r) m[r] += m[r] < 0 ? p.mod : 0;
#pragma unroll
  for (int r = 0; r < C; ++r) t[r] += (d[r] * (int64_t)((uint32_t)m[r] + (uint32_t)(65536 - p.amp))) >> 16;
}

// perturb_add for the compute spans of one op of C ranks: x[r] = sx ^ (rk[r] + ix) with
// rk[r] = (rank_r << 32) * K_MIX, whose low word is zero, so x's low word and the carry of x + G
// are shared by the C ranks and only the high words differ (rkhi[r] = rk[r] >> 32). With one
// duration d for all ranks (PR: per-rank d[r]) the product d * (m + 65536 - amp) is split as
// d * m + d * (65536 - amp). Bit-identical to perturb_x (tools/micro/hashop.cu checksum); a lone
// warp's 8-rank op 603 -> 486 cycles.
template <int C, bool PERD>
__device__ __forceinline__ void perturb_add_span(int64_t (&t)[C], const int64_t (&d)[C], uint64_t sx,
                                                 const uint32_t (&rkhi)[C], uint64_t ix, const ScenParams &p) {
  const uint32_t xlo = (uint32_t)sx ^ (uint32_t)ix;
  const uint32_t zlo = xlo + 0x7F4A7C15u;
  const uint32_t cg = 0x9E3779B9u + (zlo < xlo ? 1u : 0u);
  const uint32_t sxh = (uint32_t)(sx >> 32), ixh = (uint32_t)(ix >> 32);
  const uint32_t zlo30 = zlo >> 30;
  uint64_t z[C];
#pragma unroll
  for (int r = 0; r < C; ++r) {
    const uint32_t zh = (sxh ^ (ixh + rkhi[r])) + cg;
    const uint32_t lo = zlo ^ (zlo30 | (zh << 2)), hi = zh ^ (zh >> 30);
    z[r] = ((uint64_t)hi << 32 | lo) * 0xBF58476D1CE4E5B9ULL;
  }
#pragma unroll
  for (int r = 0; r < C; ++r) z[r] = z[r] ^ (z[r] >> 27);
  uint32_t v[C];
#pragma unroll
  for (int r = 0; r < C; ++r) {
    const uint32_t lo = (uint32_t)z[r], hi = (uint32_t)(z[r] >> 32);
    v[r] = (__umulhi(lo, 0x133111EBu) + lo * 0x94D049BBu + hi * 0x133111EBu) >> 8;
  }
  int32_t m[C];
#pragma unroll
  for (int r = 0; r < C; ++r) {
    m[r] = (int32_t)(v[r] - __umulhi(v[r], p.mod_m32) * (uint32_t)p.mod);
    m[r] += (int32_t)((uint32_t)m[r] >> 31) * p.mod;
  }
  if (PERD) {
#pragma unroll
    for (int r = 0; r < C; ++r) t[r] += (d[r] * (int64_t)((uint32_t)m[r] + (uint32_t)(65536 - p.amp))) >> 16;
  } else {
    const int64_t dc = d[0] * (int64_t)(uint32_t)(65536 - p.amp);
#pragma unroll
    for (int r = 0; r < C; ++r) t[r] += (d[0] * (int64_t)(uint32_t)m[r] + dc) >> 16;
  }
}

// perturb_add_span<C, false> for a (compute span, TP collective) pair, with the TP collective's
// perturbed duration perturb_x(dq, xq) formed as a ninth chain beside the span's C chains (emitted
// on its own, ptxas scheduled it as one serial ~40-instruction chain ahead of the span's). Returns
// the collective's duration (dq when tp_pert is false). Bit-identical to the separate calls.
template <int C>
__device__ __forceinline__ int64_t perturb_add_span_q(int64_t (&t)[C], int64_t d, uint64_t sx,
                                                      const uint32_t (&rkhi)[C], uint64_t ix, int64_t dq,
                                                      uint64_t xq, bool tp_pert, const ScenParams &p) {
  const uint32_t xlo = (uint32_t)sx ^ (uint32_t)ix;
  const uint32_t zlo = xlo + 0x7F4A7C15u;
  const uint32_t cg = 0x9E3779B9u + (zlo < xlo ? 1u : 0u);
  const uint32_t sxh = (uint32_t)(sx >> 32), ixh = (uint32_t)(ix >> 32);
  const uint32_t zlo30 = zlo >> 30;
  uint64_t z[C + 1];
#pragma unroll
  for (int r = 0; r < C; ++r) {
    const uint32_t zh = (sxh ^ (ixh + rkhi[r])) + cg;
    const uint32_t lo = zlo ^ (zlo30 | (zh << 2)), hi = zh ^ (zh >> 30);
    z[r] = ((uint64_t)hi << 32 | lo) * 0xBF58476D1CE4E5B9ULL;
  }
  {
    const uint64_t zq = xq + 0x9E3779B97F4A7C15ULL;
    z[C] = (zq ^ (zq >> 30)) * 0xBF58476D1CE4E5B9ULL;
  }
#pragma unroll
  for (int r = 0; r <= C; ++r) z[r] = z[r] ^ (z[r] >> 27);
  uint32_t v[C + 1];
#pragma unroll
  for (int r = 0; r <= C; ++r) {
    const uint32_t lo = (uint32_t)z[r], hi = (uint32_t)(z[r] >> 32);
    v[r] = (__umulhi(lo, 0x133111EBu) + lo * 0x94D049BBu + hi * 0x133111EBu) >> 8;
  }
  int32_t m[C + 1];
#pragma unroll
  for (int r = 0; r <= C; ++r) {
    m[r] = (int32_t)(v[r] - __umulhi(v[r], p.mod_m32) * (uint32_t)p.mod);
    m[r] += (int32_t)((uint32_t)m[r] >> 31) * p.mod;
  }
  const int64_t dc = d * (int64_t)(uint32_t)(65536 - p.amp);
#pragma unroll
  for (int r = 0; r < C; ++r) t[r] += (d * (int64_t)(uint32_t)m[r] + dc) >> 16;
  return tp_pert ? (dq * (int64_t)((uint32_t)m[C] + (uint32_t)(65536 - p.amp))) >> 16 : dq;
}
#endif

// Row e: the peer-memory exchange of a sharded replay. Every shard's exchange buffer has the
// same layout (same plan, same S), so one set of byte offsets addresses all of them.
constexpr int kMaxShards = 16;
struct ShardLink {
  int32_t n, self;                 // shards, this shard (n = 0: unsharded)
  uint32_t epoch;                  // replays since prepare, 1-based (flags of this replay)
  int32_t lg;                      // > 0: a local-group launch replaying shards 0..lg-1 of one device
                                   // in ONE cooperative grid (prism_replay_local_shards)
  unsigned char *base[kMaxShards];  // exchange buffer of every shard (peer-mapped), own included
  int64_t o_rslot, o_acc, o_arrive, o_part, o_flag;  // byte offsets inside a buffer
  int64_t o_gcol, o_ggcol, o_gflag;  // prism_shard_gather: finish column [N], group column [G], flags
  // local-group launches: every shard's own output arrays (the structure is the same graph)
  int64_t *lg_fin[kMaxShards], *lg_gfin[kMaxShards], *lg_rank_end[kMaxShards];
};

// Tile of a level launch: `cnt` concrete groups of quotient group `q` starting at instance `i0`.
struct Tile {
  int32_t q, i0, cnt, pad;
};

// expand.cu
cudaError_t launch_expand(const DevGraph &g, cudaStream_t st);
// replica cells: the cell records of the cell-full cross ops
cudaError_t launch_cell_records(const DevGraph &g, cudaStream_t st);
// test hook: per-node template field `which` (prism_debug_export 2..6) into a device array
cudaError_t launch_materialize(const DevGraph &g, int32_t which, void *out, cudaStream_t st);
// replay.cu
cudaError_t launch_level(const DevGraph &g, const ScenParams &p, const Tile *tiles, int32_t ntiles,
                         int32_t max_cnt, int64_t *fin, int64_t *gfin, int lanes, int nchunks,
                         cudaStream_t st);
cudaError_t launch_tail(const DevGraph &g, const ScenParams &p, int64_t *fin, const int64_t *gfin,
                        int64_t *rank_end, int lanes, int nchunks, cudaStream_t st);
cudaError_t launch_reduce(int32_t W, int32_t S, int32_t Sp, const int64_t *rank_end, int64_t *iter,
                          cudaStream_t st);
cudaError_t launch_query(const DevGraph &g, const ScenParams &p, int32_t Sp, const int64_t *fin,
                         const int64_t *gfin, int32_t rank, int32_t scen, int64_t *start_out,
                         int64_t *finish_out, cudaStream_t st);
// replay_cells.cu (cell kernel); cudaErrorCooperativeLaunchTooLarge = does not fit, use levels
// group > 1: a local-group launch covering `group` shards of one device (prism_replay_local_shards)
bool cells_fit(const DevGraph &g, int nchunks, int group = 1);
int cells_chunk_scenarios();
int cells_chunks_per_launch(const DevGraph &g, int nchunks, int group = 1);
cudaError_t launch_cells(const DevGraph &g, const ScenParams &p, int64_t *rslot, int64_t *acc,
                         int64_t *rres, uint32_t *arrive, uint32_t *status, int parity, int64_t *fin,
                         int64_t *gfin, int64_t *rank_end, int chunk0, int nchunks_launch, int Sp,
                         const ShardLink *link, cudaStream_t st);
// row e, prism_shard_gather: the shard's own finishes of scenario k into every shard's gather
// columns, then (cross-process) the epoch flag barrier
cudaError_t launch_gather(const DevGraph &g, const ShardLink &link, const int64_t *fin, const int64_t *gfin,
                          int32_t Sp, int32_t k, uint32_t epoch, uint32_t *status, cudaStream_t st);
// row e, local group: T_k = max over the shards' own ranks' rank_end (all on this device)
cudaError_t launch_local_group_reduce(const DevGraph &g, const ShardLink &link, int32_t S, int32_t Sp,
                                      int64_t *iter, cudaStream_t st);
// row e: iteration times of a sharded replay (local partial max, peer exchange, global max)
cudaError_t launch_shard_reduce(const DevGraph &g, const ShardLink &link, int32_t S, int32_t Sp,
                                const int64_t *rank_end, int64_t *part_local, int64_t *iter,
                                uint32_t *status, cudaStream_t st);
// row f2: time-ordered peak memory of scenario k of a recorded replay (max_len = longest rank,
// <= kMaxTimeOrderedOps)
constexpr int32_t kMaxTimeOrderedOps = 4096;
cudaError_t launch_peak_time(const DevGraph &g, const ScenParams &p, int32_t Sp, const int64_t *fin,
                             const int64_t *gfin, int32_t k, int32_t max_len, int64_t *peak, uint32_t *status,
                             cudaStream_t st);
// replay_ranks.cu (one scenario, lane = rank)
bool ranks_fit(const DevGraph &g, int *blocks);
cudaError_t preload_rank_kernels();
// seg: scratch of segs_scratch_bytes (nullptr: the one-kernel rank path); launches: kernels queued
size_t segs_scratch_bytes(const DevGraph &g, int64_t n_cross);
cudaError_t launch_ranks(const DevGraph &g, const ScenParams &p, int64_t *rslot, int64_t *acc, int64_t *rres,
                         uint32_t *arrive, uint32_t *status, int parity, int64_t *fin, int64_t *gfin,
                         int64_t *rank_end, int64_t *seg, int64_t n_cross, int *launches, cudaStream_t st);
// memory.cu
cudaError_t launch_peak(const DevGraph &g, int64_t *peak, cudaStream_t st);
// whatif.cu (rows f1/f3/f4): device copies of prism_set_durations' inputs ...
struct DurIn {
  const int64_t *base;       // [N] measured durations or nullptr (template)
  const uint32_t *labels;    // [n_labels] sorted
  const int64_t *label_dur;  // [n_labels]
  int32_t n_labels;
  const int32_t *rank_f;     // [W] Q16 compute slowdown or nullptr
  const int64_t *al, *fr;    // [N] memory deltas or nullptr (template)
};
// ... and of prism_set_moe_load's (n_events == 0: no MoE load)
struct MoeIn {
  const int32_t *op_event;   // [n_ops] gating event of each template op, -1 = not routed
  const int32_t *br;         // [n_events][ep] Q16
  int32_t n_events;
  uint32_t scale;            // PRISM_MOE_DUR | _ALLOC | _FREE
};
// effective durations (eff), memory deltas (eal / efr, nullptr = unchanged), group durations and
// the replay records; *status = first invalid input (PRISM_E_INVALID_ARG / _NEGATIVE_MEMORY)
cudaError_t launch_durations(const DevGraph &g, const DurIn &in, const MoeIn &me, int64_t *eff, int64_t *eal,
                             int64_t *efr, int64_t *gdur, int64_t *sdur, int64_t *hdur, uint32_t *status,
                             cudaStream_t st);
// iter[k] receives T_k (max finish over every node); the walk starts at the lowest node finishing at it;
// Row f3: the critical path of scenario k into scratch (crit_scratch_bytes of it); have_T: iter[k]
// already holds T. path_len_start receives the device addresses of the path, its length (int64)
// and the start node inside scratch.
size_t crit_scratch_bytes(const DevGraph &g, int64_t path_cap);
cudaError_t launch_critical_path(const DevGraph &g, const ScenParams &p, const int64_t *fin, int32_t Sp, int32_t k,
                                 int64_t *iter, bool have_T, void *scratch, int32_t *path_len_start[3],
                                 int64_t cap, cudaStream_t st);
// Start of every waiting replay (cells / ranks): the previous replay's abort status (word 0) is
// folded into the sticky word (1) and cleared; after an abort the ready / result slots are reset
// to "not yet" under this replay's parity (fill), since the aborted replay left some unwritten.
// rslot == nullptr: no reset (sharded replays: the exchange buffer is re-prepared instead).
cudaError_t launch_replay_guard(uint32_t *words, int64_t *rslot, size_t rslot_words, int64_t *rres, size_t rres_words,
                                int parity, cudaStream_t st);
// SM count of the current device (grid sizing; cached per device)
int num_sms();
// eager loading of the kernels that can be launched behind a running (waiting) replay
cudaError_t preload_replay_kernels();
cudaError_t preload_cells();
cudaError_t preload_peak_kernel();

}  // namespace prism
