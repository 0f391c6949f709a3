// replay_ranks.cu — the single-scenario replay (rows a6-a8 at S = 1).
//
// Same semantics as the cell kernel (readings Z2-Z5), laid out
// for ONE scenario, where lane = scenario would leave 31 lanes idle. Two forms:
//   * the segment path (below, segs_ok: tp <= 8, no replica / EP-CTA plan): a parallel walk of
//     every segment between cross-warp ops (max-plus summaries), a cooperative chain kernel that
//     only performs the cross-warp rendezvous (lane = rank), and a parallel walk writing every
//     op's finish;
//   * the rank kernel (fallback): a warp owns 32 ranks of one pipeline stage (tp_i fastest, then
//     dp_i; they all run the stage template), one per lane, and walks every op:
//       compute span      : t += dur'(own rank)
//       TP collective     : segmented max over the tp lanes of the lane's TP group (xor
//                           shuffles, tp a power of two) + the group's dur'
//       chained collective: t += dur'(own group) (every member sits at the previous
//                           occurrence's shared finish, reading of plan.cpp)
//       cross-warp group  : cross_sync below.
// Template records are broadcast to the lanes from a 32-op batch loaded one batch ahead; cross-op
// slot records are loaded one cross op ahead. Every warp of a chain / rank launch is co-resident
// (cooperative launch) and a %globaltimer watchdog turns any stall into PRISM_E_DEADLOCK.
#include <cuda_runtime.h>

#include <algorithm>

#include "graph.h"

namespace prism {

namespace {

constexpr uint64_t K_GOLD = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t K_MIX = 0xBF58476D1CE4E5B9ULL;
constexpr int kMaxSlots = 4;  // P2P nodes batch at most 4 messages

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int64_t ldr64(const int64_t *p) {
  int64_t v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ldr32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void str64(int64_t *p, int64_t v) {
  asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct RankArgs {
  int64_t *rslot;    // [M_cross] ready slots (parity-encoded)
  int64_t *acc;      // [G_large] max accumulators (zeroed per replay)
  int64_t *rres;     // [G_large] result slots (parity-encoded)
  uint32_t *arrive;  // [G_large] arrival counters (zeroed per replay)
  uint32_t *status;
  uint64_t timeout_ns;
  int32_t parity;
  int32_t per_warp_dp;  // dp coordinates per warp (32 / tp)
  int32_t warps_per_stage;
};

// group id (uid bits 24..55) of a rank's TP / DP / EP / EDP / WORLD group (closed form, row a2)
__device__ __forceinline__ uint64_t coll_gid(const DevGraph &g, uint32_t type, int32_t s, int32_t tpi, int32_t dpi) {
  const int32_t epi = dpi % g.ep, edpi = dpi / g.ep;
  switch (type) {
    case PRISM_ROLE_TP: return (uint64_t)s + (uint64_t)g.pp * dpi;
    case PRISM_ROLE_DP: return (uint64_t)tpi + (uint64_t)g.tp * s;
    case PRISM_ROLE_EP: return (uint64_t)tpi + (uint64_t)g.tp * (s + (uint64_t)g.pp * edpi);
    case PRISM_ROLE_EDP: return (uint64_t)tpi + (uint64_t)g.tp * (s + (uint64_t)g.pp * epi);
    default: return 0;  // WORLD
  }
}

// The slot records of one cross-warp op of a rank (<= kMaxSlots groups).
struct XRec {
  int32_t h0, ns;
  uint32_t meta[kMaxSlots];
  int32_t hb[kMaxSlots];
  int64_t dur[kMaxSlots];
  uint64_t uid[kMaxSlots];
  int32_t grp[kMaxSlots];  // batched P2P nodes (ns > 1): each group's id, for its finish in gfin
};
__device__ __forceinline__ void load_xrec(const DevGraph &g, XRec &x, int32_t h0, int32_t ns) {
  x.h0 = h0;
  x.ns = ns;
#pragma unroll
  for (int q = 0; q < kMaxSlots; ++q) {
    x.meta[q] = 0;
    x.hb[q] = 0;
    x.dur[q] = 0;
    x.uid[q] = 0;
    x.grp[q] = 0;
    if (q < ns) {
      x.meta[q] = g.h_meta[h0 + q];
      x.hb[q] = g.h_base[h0 + q];
      x.dur[q] = g.h_dur[h0 + q];
      x.uid[q] = g.h_uid[h0 + q];
      // loaded with the rest (one cross op ahead): the finish's gfin store then waits for no load
      if (ns > 1) x.grp[q] = g.node_grp[h0 + q];
    }
  }
}

// Cross-warp synchronization of one rank at ready time t: the lane deposits t into its own ready
// slot of each group (value-as-flag, parity-encoded; a large group: red.max + acq_rel arrival, the
// completing member publishes the max in a result slot), polls its partners, and returns the
// node's finish = max over its groups of (start + dur') in *out. False: the replay was aborted
// (another warp's watchdog, or this one's).

__device__ __forceinline__ bool cross_sync(const DevGraph &g, const ScenParams &p, const RankArgs &a, const XRec &x,
                                           int64_t t, uint64_t sx, bool gpert, bool ppert, int64_t *gfin,
                                           int64_t *out) {
  const int64_t pm = a.parity ? -1 : 0;
  int64_t val[kMaxSlots];
  uint32_t pend = 0;
#pragma unroll
  for (int q = 0; q < kMaxSlots; ++q) {
    val[q] = t;
    if (q < x.ns) {
      pend |= 1u << q;
      if (!(x.meta[q] & 0x80000000u)) {
        str64(a.rslot + x.hb[q] + (int32_t)((x.meta[q] >> 16) & 0x7FFF), t ^ pm);
      } else {  // large group: accumulate, arrive; the completing member publishes the max
        asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(a.acc + x.hb[q]), "l"((uint64_t)t) : "memory");
        uint32_t old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.arrive + x.hb[q]) : "memory");
        if (old + 1 == (x.meta[q] & 0xFFFF)) {
          val[q] = ldr64(a.acc + x.hb[q]);
          str64(a.rres + x.hb[q], val[q] ^ pm);
          pend &= ~(1u << q);
        }
      }
    }
  }
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (true) {
#pragma unroll
    for (int q = 0; q < kMaxSlots; ++q) {
      if (!((pend >> q) & 1u)) continue;
      bool ok = true;
      int64_t m = val[q];
      if (x.meta[q] & 0x80000000u) {
        const int64_t v = ldr64(a.rres + x.hb[q]) ^ pm;
        ok = v >= 0;
        m = max(m, v);
      } else {
        const int32_t size = (int32_t)(x.meta[q] & 0xFFFF), own = (int32_t)((x.meta[q] >> 16) & 0x7FFF);
        for (int32_t mm = 0; mm < size; ++mm) {
          if (mm == own) continue;
          const int64_t v = ldr64(a.rslot + x.hb[q] + mm) ^ pm;
          ok &= v >= 0;
          m = max(m, v);
        }
      }
      if (ok) {
        val[q] = m;
        pend &= ~(1u << q);
      }
    }
    if (__all_sync(0xffffffffu, pend == 0)) break;
    ++spins;
    // short sleeps: a replay of one scenario is a chain of handoffs, each one's latency is the
    // poll interval (few warps poll, so L2 polling traffic is no concern)
    if (spins > 32) __nanosleep(spins > 512 ? 1024u : 64u);
    if ((spins & 63) == 0) {
      if (ldr32(a.status) != 0) return false;
      if (t0 == 0) t0 = gtimer();
      if (gtimer() - t0 > a.timeout_ns) {
        atomicCAS(a.status, 0u, (uint32_t)PRISM_E_DEADLOCK);
        return false;
      }
    }
  }
  int64_t fr = 0;
#pragma unroll
  for (int q = 0; q < kMaxSlots; ++q) {
    if (q >= x.ns) continue;
    int64_t gd = x.dur[q];
    const uint64_t uid = x.uid[q];
    const bool pr = (uid >> 56) == PRISM_ROLE_P2P ? ppert : gpert;
    if (pr) gd = perturb_x(gd, sx ^ (uid * K_MIX), p);
    const int64_t f = val[q] + gd;
    fr = max(fr, f);
    if (x.ns > 1) gfin[x.grp[q]] = f;  // batched P2P groups' finishes, for queries
  }
  *out = fr;
  return true;
}

template <bool PR>
__global__ void __launch_bounds__(32, 16) rank_kernel(DevGraph g, ScenParams p, RankArgs a, int64_t *__restrict__ fin,
                                                     int64_t *__restrict__ gfin, int64_t *__restrict__ rank_end) {
  const int lane = threadIdx.x & 31;
  const int32_t w = blockIdx.x;
  if (w == g.stall_unit) return;  // watchdog test hook (prism_debug_set)
  const int32_t s = w / a.warps_per_stage;
  const int32_t tpi = lane % g.tp;
  const int32_t dpi = (w % a.warps_per_stage) * a.per_warp_dp + lane / g.tp;
  const bool active = dpi < g.dp && s < g.pp;
  const int32_t r = active ? (g.order == PRISM_ORDER_MEGATRON ? tpi + g.tp * (dpi + g.dp * s) : tpi + g.tp * (s + g.pp * dpi)) : 0;
  const int32_t rb = active ? g.rank_ptr[r] : 0;
  // fin row of op i: cell-interleaved (graph.h fin_off; one scenario: row = element), so the tp
  // lanes of a cell store op i to consecutive words
  const int64_t frow0 = active ? cell_row0(g, r) - g.fin_node0 : 0;
  const int32_t fstride = cell_row_stride(g);
  const int32_t rs = active ? g.node_gptr[rb] : 0;  // the rank's first membership slot
  const int32_t s0 = s < g.pp ? s : 0;
  const int32_t len = (int32_t)g.t_len[s0];
  const int64_t op0 = g.t_op0[s0];
  const int32_t kg = p.first;  // the replay's single scenario (perturbation key)
  const uint64_t sx = p.seed ^ ((uint64_t)kg * K_GOLD);
  const uint64_t rkx = ((uint64_t)r << 32) * K_MIX;
  const bool cpert = (p.mask & 1u) && p.amp > 0 && kg > 0;
  const bool gpert = (p.mask & 2u) && p.amp > 0 && kg > 0;
  const bool ppert = (p.mask & 4u) && p.amp > 0 && kg > 0;
  int64_t t = 0;
  // template records, one 32-op batch ahead: class | group type << 8, occurrence, duration
  uint32_t ncw = 0, nocc = 0;
  int64_t ndur = 0;
  auto load_rec = [&](int32_t i, uint32_t &cw, uint32_t &occ, int64_t &dur) {
    const int64_t op = op0 + i;
    const uint32_t c = __ldg(g.t_cls + op) & 0xFu;  // bit 0x10: (compute, TP) pair flag of the cell kernel
    const int32_t q0 = __ldg(g.t_q0 + op);
    uint32_t type = 0;
    occ = 0;
    dur = __ldg(g.t_dur + op);
    if (q0 >= 0) {
      type = (uint32_t)__ldg(&g.q[q0].type);
      occ = (uint32_t)__ldg(&g.q[q0].occ);
      dur = __ldg(&g.q[q0].dur);
    }
    cw = c | (type << 8);
  };
  if (lane < len) load_rec(lane, ncw, nocc, ndur);
  int64_t pd = (PR && active && len > 0) ? __ldg(g.node_sdur + rb) : 0;
  // the next cross-warp op of the stage (plan x_ops: class-2 ops) and its slot records, loaded
  // one cross op ahead so that a rank reaching it deposits and polls without a dependent load
  int32_t xk = g.x_ptr[s0];
  const int32_t xend = g.x_ptr[s0 + 1];
  int32_t xt = -1;
  XRec xr;
  auto prefetch_x = [&]() {
    xt = -1;
    int32_t h0 = 0, ns = 0;
    if (xk < xend) {
      const XOp xo = g.x_ops[xk];
      xt = xo.tidx;
      h0 = rs + xo.hoff;
      ns = active ? min(xo.ns, kMaxSlots) : 0;
    }
    load_xrec(g, xr, h0, ns);
  };
  prefetch_x();
  for (int32_t base = 0; base < len; base += 32) {
    const int32_t cnt = min(32, len - base);
    const uint32_t bcw = ncw, bocc = nocc;
    const int64_t bdur = ndur;
    if (base + 32 + lane < len) load_rec(base + 32 + lane, ncw, nocc, ndur);
    for (int32_t j = 0; j < cnt; ++j) {
      const int32_t i = base + j;
      const uint32_t cw = __shfl_sync(0xffffffffu, bcw, j);
      const uint32_t occ = __shfl_sync(0xffffffffu, bocc, j);
      int64_t d = __shfl_sync(0xffffffffu, bdur, j);
      const uint32_t c = cw & 0xFF, type = cw >> 8;
      if (PR) {  // this rank's own (overridden) duration
        d = pd;
        if (active && i + 1 < len) pd = __ldg(g.node_sdur + rb + i + 1);
      }
      if (c == 0) {
        t += cpert ? perturb_x(d, sx ^ (rkx + (uint64_t)i * K_MIX), p) : d;
      } else if (c == 1 || c == 3) {
        int64_t m = t;
        if (c == 1)  // TP collective: segmented max over the lane's TP group
          for (int off = 1; off < g.tp; off <<= 1) m = max(m, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)m, off));
        if (gpert) {
          const uint64_t uid = ((uint64_t)type << 56) | (coll_gid(g, type, s0, tpi, dpi) << 24) | (uint64_t)occ;
          d = perturb_x(d, sx ^ (uid * K_MIX), p);
        }
        t = m + d;
      } else {  // cross-warp synchronization: the lane's own rank, its <= 4 groups
        int64_t fr = 0;
        if (i == xt) {  // prefetched (class 2)
          if (!cross_sync(g, p, a, xr, t, sx, gpert, ppert, gfin, &fr)) return;
          ++xk;  // the next cross op's records load while the compute spans run
          prefetch_x();
        } else {  // class 4 (EP CTA ops of a replica plan): records loaded here
          XRec xl;
          const int32_t h0 = active ? g.node_gptr[rb + i] : 0;
          load_xrec(g, xl, h0, active ? g.node_gptr[rb + i + 1] - h0 : 0);
          if (!cross_sync(g, p, a, xl, t, sx, gpert, ppert, gfin, &fr)) return;
        }
        if (active) t = fr;
      }
      if (p.record && active) fin[frow0 + (int64_t)i * fstride] = t;
    }
  }
  if (active) rank_end[r] = t;
}


// ---- the segment path: S = 1 in three launches ---------------------------------------------
//
// Between two cross-warp ops a rank's ops only add durations (compute spans, chained
// collectives) or take the max over the cell's tp ranks (TP collectives), so a cell's times over
// such a SEGMENT are a max-plus function of its ranks' start times s_r of a fixed shape: before
// the segment's first TP collective t_r = s_r + A_r; from it on every rank is at
// T = max_r (s_r + pre_r) + dT plus a rank-independent-start offset B_r. Durations (and their
// perturbations) do not depend on the start times, so:
//   1. seg_walk_kernel<summary>: every (stage, segment, dp cell) in parallel, a lane per cell
//      holding its tp ranks in registers (the cells of a stage run one template: convergent
//      warps): (flag, dT, pre_r, end_r) of the segment, computed from zero starts;
//   2. seg_chain_kernel (cooperative, lane = rank as the rank kernel): only the cross-warp ops,
//      each rank's ready time = flag ? max over its TP lanes (s_r + pre_r) + dT + end_r
//      : s_r + end_r, then the rendezvous (cross_sync); it records each segment's start s_r and
//      the cross ops' finishes;
//   3. seg_walk_kernel<fin> (record only): every segment again from its recorded starts, writing
//      the finish of every op.
// The chain of dependent steps is then one per cross op instead of one per op (~16x shorter on
// C5), and the per-op work runs at full occupancy.
// Layout: segment g = x_ptr[s] + s + j (j = 0 .. nx_s; segment j ends before cross op j, the last
// one at the template's end); summ[(g * F + field) * dp + dp_i] with F = 2 tp + 2 fields
// (flag, dT, pre[tp], end[tp]); sstart[(g * tp + tp_i) * dp + dp_i].

// Lane = (cell, rank): a warp holds 32 / C cells of one stage's segment, C consecutive lanes per
// cell, so a TP collective is a C-lane xor-shuffle max, each lane hashes only its own rank, and
// op i's finishes of a cell are C consecutive words (one coalesced store per op). Template
// records come 32 ops per round trip (lane l loads op i0 + base + l, broadcast by shuffles), the
// next batch in flight.
template <int C, bool PR, bool FIN>
__global__ void __launch_bounds__(128) seg_walk_kernel(DevGraph g, ScenParams p, int64_t *__restrict__ summ,
                                                       const int64_t *__restrict__ sstart, int64_t *__restrict__ fin,
                                                       int32_t nsegs, int32_t dchunks) {
  constexpr int CPW = 32 / C;  // cells per warp
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (wid >= (int64_t)nsegs * dchunks) return;  // whole warps only
  const int32_t gs = (int32_t)(wid / dchunks), chunk = (int32_t)(wid % dchunks);
  // the segment's stage: the last s whose first segment x_ptr[s] + s is <= gs. pp <= 32: one
  // coalesced load of x_ptr and a ballot (the scan below costs a dependent round trip per stage)
  int32_t s = 0, xs, nx;
  if (g.pp <= 31) {
    const int32_t xv = lane <= g.pp ? g.x_ptr[lane] + lane : 0x7FFFFFFF;
    const uint32_t m = __ballot_sync(0xffffffffu, lane < g.pp && xv <= gs);
    s = 31 - __clz((int)m);
    xs = __shfl_sync(0xffffffffu, xv, s) - s;
    nx = __shfl_sync(0xffffffffu, xv, s + 1) - (s + 1) - xs;
  } else {
    while (s + 1 < g.pp && g.x_ptr[s + 1] + s + 1 <= gs) ++s;
    xs = g.x_ptr[s];
    nx = g.x_ptr[s + 1] - xs;
  }
  const int32_t j = gs - xs - s;
  const int32_t len = (int32_t)g.t_len[s];
  const int32_t i0 = j == 0 ? 0 : g.x_ops[xs + j - 1].tidx + 1;
  const int32_t i1 = j < nx ? g.x_ops[xs + j].tidx : len;
  const int32_t rr = lane % C;                   // rank of the cell (tp_i)
  const int32_t dpi = chunk * CPW + lane / C;    // the cell's dp coordinate
  const bool active = dpi < g.dp;                // inactive lanes run along (shuffles), store nothing
  const int32_t dpc = active ? dpi : 0;
  const int32_t r0 = dg_rank_of(g, 0, s, dpc), rank = r0 + rr;
  const int32_t kg = p.first;
  const uint64_t sx = p.seed ^ ((uint64_t)kg * K_GOLD);
  const bool cpert = (p.mask & 1u) && p.amp > 0 && kg > 0;
  const bool gpert = (p.mask & 2u) && p.amp > 0 && kg > 0;
  const uint64_t rkx = ((uint64_t)rank << 32) * K_MIX;
  const int32_t rb = PR ? g.rank_ptr[rank] : 0, rb0 = PR ? g.rank_ptr[r0] : 0;
  int64_t t = (FIN && j > 0 && active) ? sstart[((int64_t)gs * C + rr) * g.dp + dpi] : 0;
  int64_t pre = 0, dT = 0;
  bool tp_seen = false;
  const int64_t top0 = g.t_op0[s];
  int64_t *fp = fin + (cell_row0(g, r0) - g.fin_node0) + (int64_t)i0 * C + rr;
  // the cell's group uid base for the TP / chained collectives (closed form, row a2)
  auto cell_uid = [&](uint64_t qi) {
    return group_uid_packed(g, qi, group_inst(g, (int32_t)(qi & 0xFF), 0, dpc, dpc % g.ep, dpc / g.ep));
  };
  uint32_t ncls = 0;
  int64_t nd = 0;
  uint64_t nqi = 0;
  auto load_rec = [&](int32_t i, uint32_t &c, int64_t &d, uint64_t &qi) {
    const int64_t op = top0 + i;
    c = __ldg(g.t_cls + op) & 0xFu;
    d = __ldg(g.t_sdur + op);
    qi = (c == 1 || c == 3) ? __ldg(g.t_qinfo + op) : 0;
  };
  if (i0 + lane < i1) load_rec(i0 + lane, ncls, nd, nqi);
  for (int32_t base = i0; base < i1; base += 32) {
    const int32_t cnt = min(32, i1 - base);
    const uint32_t bc = ncls;
    const int64_t bd = nd;
    const uint64_t bq = nqi;
    if (base + 32 + lane < i1) load_rec(base + 32 + lane, ncls, nd, nqi);
    for (int32_t jj = 0; jj < cnt; ++jj) {
      const int32_t i = base + jj;
      const uint32_t c = __shfl_sync(0xffffffffu, bc, jj);
      int64_t d = __shfl_sync(0xffffffffu, bd, jj);
      // PR: own duration for compute spans and chained collectives; a TP collective's record
      // duration is the group's (every member's node carries it; rank 0's is read)
      const int64_t dr = PR ? __ldg(g.node_sdur + (c == 1 ? rb0 : rb) + i) : d;
      if (c == 0) {  // compute span
        t += cpert ? perturb_x(dr, sx ^ (rkx + (uint64_t)i * K_MIX), p) : dr;
      } else {
        const uint64_t qi = __shfl_sync(0xffffffffu, bq, jj);
        if (c == 1) {  // TP collective of the cell: max over its C lanes + the group's dur'
          int64_t m = t;
#pragma unroll
          for (int off = 1; off < C; off <<= 1) m = max(m, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)m, off));
          const int64_t dd = gpert ? perturb_x(dr, sx ^ (cell_uid(qi) * K_MIX), p) : dr;
          if (!FIN && !tp_seen) {  // summary: the first fixes pre_r and dT; later times are relative to T
            tp_seen = true;
            dT = dd;
            pre = t;
            t = 0;
          } else {
            t = m + dd;
          }
        } else {  // chained collective (c == 3): every member starts at its own ready time;
                  // rank r's group: gid steps by 1 per tp_i (DP / EP / EDP), one group for WORLD
          if (gpert) {
            const uint64_t ux = cell_uid(qi);
            const uint64_t step = (ux >> 56) == PRISM_ROLE_WORLD ? 0ull : (1ull << 24);
            t += perturb_x(dr, sx ^ ((ux + (uint64_t)rr * step) * K_MIX), p);
          } else {
            t += dr;
          }
        }
      }
      if (FIN) {
        if (active) fp[0] = t;
        fp += C;
      }
    }
  }
  if (!FIN && active) {
    int64_t *o = summ + (int64_t)gs * (2 * C + 2) * g.dp + dpi;
    if (rr == 0) {
      o[0] = tp_seen ? 1 : 0;
      o[(int64_t)g.dp] = dT;
    }
    o[(int64_t)(2 + rr) * g.dp] = pre;
    o[(int64_t)(2 + C + rr) * g.dp] = t;
  }
}

__global__ void __launch_bounds__(32, 16) seg_chain_kernel(DevGraph g, ScenParams p, RankArgs a,
                                                           const int64_t *__restrict__ summ,
                                                           int64_t *__restrict__ sstart, int64_t *__restrict__ fin,
                                                           int64_t *__restrict__ gfin, int64_t *__restrict__ rank_end) {
  const int lane = threadIdx.x & 31;
  const int32_t w = blockIdx.x;
  if (w == g.stall_unit) return;  // watchdog test hook (prism_debug_set)
  const int32_t s = w / a.warps_per_stage, chunk = w % a.warps_per_stage;
  const int32_t tp = g.tp, tpi = lane % tp;
  const int32_t dpi = chunk * a.per_warp_dp + lane / tp;
  const bool active = dpi < g.dp && s < g.pp;
  const int32_t r = active ? dg_rank_of(g, tpi, s, dpi) : 0;
  const int32_t rb = active ? g.rank_ptr[r] : 0;
  const int64_t frow0 = active ? cell_row0(g, r) - g.fin_node0 : 0;
  const int32_t fstride = cell_row_stride(g);
  const int32_t rs = active ? g.node_gptr[rb] : 0;
  const int32_t s0 = s < g.pp ? s : 0;
  const int32_t dpc = active ? dpi : 0;
  const int32_t kg = p.first;
  const uint64_t sx = p.seed ^ ((uint64_t)kg * K_GOLD);
  const bool gpert = (p.mask & 2u) && p.amp > 0 && kg > 0;
  const bool ppert = (p.mask & 4u) && p.amp > 0 && kg > 0;
  const int32_t xs = g.x_ptr[s0], nx = g.x_ptr[s0 + 1] - xs;
  const int64_t F = 2 * tp + 2, dp = g.dp;
  // segment summaries and cross-op records, one cross op ahead
  auto load_sum = [&](int32_t j, int64_t &fl, int64_t &dT, int64_t &pre, int64_t &end) {
    const int64_t *o = summ + (int64_t)(xs + s0 + j) * F * dp + dpc;
    fl = o[0];
    dT = o[dp];
    pre = o[(2 + tpi) * dp];
    end = o[(2 + tp + tpi) * dp];
  };
  XRec xr, xn;  // this cross op's records and the next one's (loaded a rendezvous ahead)
  int32_t ti = 0, tn = 0;  // their template indices
  // the slot records of op j are addressed by its XOp entry, which is loaded one rendezvous
  // earlier still (xq): loading both at once made the warp wait for the entry before its deposit
  XOp xq{0, 0, 0, 0};
  auto load_x = [&](int32_t j, const XOp &xo, XRec &x, int32_t &ti_) {
    int32_t h0 = 0, ns = 0;
    ti_ = 0;
    if (j < nx) {
      h0 = rs + xo.hoff;
      ns = active ? min(xo.ns, kMaxSlots) : 0;
      ti_ = xo.tidx;
    }
    load_xrec(g, x, h0, ns);
  };
  int64_t fl, dT, pre, end;
  load_sum(0, fl, dT, pre, end);
  if (0 < nx) xq = g.x_ops[xs];
  load_x(0, xq, xn, tn);
  if (1 < nx) xq = g.x_ops[xs + 1];
  int64_t t = 0;  // the current segment's start s_r
  for (int32_t j = 0; j <= nx; ++j) {
    int64_t m = t + pre;
    for (int off = 1; off < tp; off <<= 1) m = max(m, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)m, off));
    const int64_t ready = fl ? m + dT + end : t + end;
    if (j == nx) {
      if (active) rank_end[r] = ready;
      break;
    }
    xr = xn;
    ti = tn;
    const int32_t i = ti;
    // the next segment's summary and cross op records load during this rendezvous, and the XOp
    // entry of the op after
    load_sum(j + 1, fl, dT, pre, end);
    load_x(j + 1, xq, xn, tn);
    if (j + 2 < nx) xq = g.x_ops[xs + j + 2];
    int64_t fr = 0;
    if (!cross_sync(g, p, a, xr, ready, sx, gpert, ppert, gfin, &fr)) return;
    t = fr;
    if (active && p.record) {
      fin[frow0 + (int64_t)i * fstride] = fr;
      sstart[((int64_t)(xs + s0 + j + 1) * tp + tpi) * dp + dpi] = fr;
    }
  }
}
}  // namespace

// Usable when: one scenario, unsharded, single-stream, tp a power of two <= 32.
bool ranks_fit(const DevGraph &g, int *blocks) {
  if (g.n_shards > 1 || g.ms || g.tp > 32 || (g.tp & (g.tp - 1))) return false;
  const int32_t per_warp_dp = 32 / g.tp;
  const int64_t wps = (g.dp + per_warp_dp - 1) / per_warp_dp;
  const int64_t need = wps * g.pp;
  int dev = 0, sms = 0, per_sm = 0, coop = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  const void *fn = g.per_rank_dur ? (const void *)rank_kernel<true> : (const void *)rank_kernel<false>;
  if (!coop || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32, 0) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  int per_sm2 = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, (const void *)seg_chain_kernel, 32, 0) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  per_sm = std::min(per_sm, per_sm2);
  if (blocks) *blocks = (int)need;
  return need >= 1 && (int64_t)per_sm * sms >= need;
}

cudaError_t preload_rank_kernels() {
  cudaFuncAttributes at;
  cudaError_t e = cudaFuncGetAttributes(&at, (const void *)rank_kernel<false>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&at, (const void *)rank_kernel<true>);
  return e;
}

// The segment path applies to plans whose cross-warp ops are exactly the x_ops list (no EP-CTA
// ops) with one-rank-per-lane TP cells of width <= 8 (cell_R <= 1).
bool segs_ok(const DevGraph &g) { return g.cta_ks <= 1 && g.cell_R <= 1 && g.tp <= 8; }

size_t segs_scratch_bytes(const DevGraph &g, int64_t n_cross) {
  const int64_t nsegs = n_cross + g.pp;
  return (size_t)nsegs * (size_t)(3 * g.tp + 2) * (size_t)g.dp * 8;
}

template <int C>
static cudaError_t launch_walk(const DevGraph &g, const ScenParams &p, int64_t *summ, const int64_t *sstart,
                               int64_t *fin, int32_t nsegs, bool finpass, cudaStream_t st) {
  const int32_t dchunks = (g.dp + 32 / C - 1) / (32 / C);
  const int64_t warps = (int64_t)nsegs * dchunks;
  const unsigned blocks = (unsigned)((warps + 3) / 4);
  if (blocks == 0) return cudaSuccess;
  if (finpass) {
    if (g.per_rank_dur) seg_walk_kernel<C, true, true><<<blocks, 128, 0, st>>>(g, p, summ, sstart, fin, nsegs, dchunks);
    else seg_walk_kernel<C, false, true><<<blocks, 128, 0, st>>>(g, p, summ, sstart, fin, nsegs, dchunks);
  } else {
    if (g.per_rank_dur) seg_walk_kernel<C, true, false><<<blocks, 128, 0, st>>>(g, p, summ, sstart, fin, nsegs, dchunks);
    else seg_walk_kernel<C, false, false><<<blocks, 128, 0, st>>>(g, p, summ, sstart, fin, nsegs, dchunks);
  }
  return cudaGetLastError();
}

static cudaError_t launch_walk_tp(const DevGraph &g, const ScenParams &p, int64_t *summ, const int64_t *sstart,
                                  int64_t *fin, int32_t nsegs, bool finpass, cudaStream_t st) {
  switch (g.tp) {
    case 1: return launch_walk<1>(g, p, summ, sstart, fin, nsegs, finpass, st);
    case 2: return launch_walk<2>(g, p, summ, sstart, fin, nsegs, finpass, st);
    case 4: return launch_walk<4>(g, p, summ, sstart, fin, nsegs, finpass, st);
    case 8: return launch_walk<8>(g, p, summ, sstart, fin, nsegs, finpass, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ranks(const DevGraph &g, const ScenParams &p, int64_t *rslot, int64_t *acc, int64_t *rres,
                         uint32_t *arrive, uint32_t *status, int parity, int64_t *fin, int64_t *gfin,
                         int64_t *rank_end, int64_t *seg, int64_t n_cross, int *launches, cudaStream_t st) {
  int blocks = 0;
  if (!ranks_fit(g, &blocks)) return cudaErrorCooperativeLaunchTooLarge;
  const int32_t per_warp_dp = 32 / g.tp;
  RankArgs a{rslot, acc, rres, arrive, status, g.watchdog_ns, parity, per_warp_dp,
             (int32_t)((g.dp + per_warp_dp - 1) / per_warp_dp)};
  DevGraph gg = g;
  ScenParams pp = p;
  if (seg && segs_ok(g)) {
    const int32_t nsegs = (int32_t)(n_cross + g.pp);
    int64_t *summ = seg, *sstart = seg + (int64_t)nsegs * (2 * g.tp + 2) * g.dp;
    cudaError_t e = launch_walk_tp(g, p, summ, sstart, fin, nsegs, false, st);
    if (e != cudaSuccess) return e;
    void *args[] = {&gg, &pp, &a, &summ, &sstart, &fin, &gfin, &rank_end};
    e = cudaLaunchCooperativeKernel((const void *)seg_chain_kernel, dim3(blocks), dim3(32), args, 0, st);
    if (e != cudaSuccess) return e;
    if (fin) e = launch_walk_tp(g, p, summ, sstart, fin, nsegs, true, st);
    if (launches) *launches = fin ? 3 : 2;
    return e;
  }
  void *args[] = {&gg, &pp, &a, &fin, &gfin, &rank_end};
  const void *fn = g.per_rank_dur ? (const void *)rank_kernel<true> : (const void *)rank_kernel<false>;
  if (launches) *launches = 1;
  return cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(32), args, 0, st);
}

}  // namespace prism
