// cell_kernel.cuh — the cell kernel template (see replay_cells.cu for what it computes).
// Included by the cells_k_*.cu instantiation units (compiled in parallel: one unit per
// (sharded, per-rank durations, multi-stream) variant) and by replay_cells.cu (launch logic).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "graph.h"

namespace prism {

namespace {

constexpr uint64_t K_GOLD = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t K_MIX = 0xBF58476D1CE4E5B9ULL;
constexpr int SC = 32;          // scenarios per unit (one warp, lane = scenario)
constexpr int WARPS = 1;        // units per CTA (1: warps spread evenly over the SMs)
constexpr int MAX_TP = 8;       // tp of the instantiated cell kernels
constexpr int kPollBatch = 8;  // poll loads issued back to back per batch (16 raised register pressure: slower)


__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int64_t ld_relaxed64(const int64_t *p) {
  int64_t v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Deposit of a ready time: a strong (relaxed, gpu-scope) store goes to L2 right away; a weak store
// may linger in the SM for tens of microseconds (measured), which the pipeline pays per handoff.
__device__ __forceinline__ void st_relaxed64(int64_t *p, int64_t v) {
  asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_max(int64_t *p, int64_t v) {
  asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"((uint64_t)v) : "memory");
}
// System-scope variants for the sharded replay (row e): the other party is a thread on a peer GPU
// reaching this memory over NVLink, so the strong operations must be scoped .sys.
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int64_t ld_relaxed_sys64(const int64_t *p) {
  int64_t v;
  asm volatile("ld.relaxed.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys64(int64_t *p, int64_t v) {
  asm volatile("st.relaxed.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_max_sys(int64_t *p, int64_t v) {
  asm volatile("red.relaxed.sys.global.max.u64 [%0], %1;" ::"l"(p), "l"((uint64_t)v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
template <bool SH>
__device__ __forceinline__ int64_t poll64(const int64_t *p) {
  return SH ? ld_relaxed_sys64(p) : ld_relaxed64(p);
}
template <bool SH>
__device__ __forceinline__ uint32_t poll32(const uint32_t *p) {
  return SH ? ld_relaxed_sys(p) : ld_relaxed(p);
}

#ifdef PRISM_CELL_STATS
__device__ unsigned long long g_dep_time[1 << 22];     // deposit globaltimer per ready slot (chunk 0)
__device__ unsigned long long g_lat[4];                // sum latency, sum skew, count, max latency
__device__ unsigned long long g_wait_hist[16 * 4096];  // [stage][template op] wait cycles (stage < 16)
__device__ unsigned long long g_cell_stats[16384 * 8];  // per warp: total, cross, -, polls, start, end
__device__ unsigned long long g_tl[16 * 128 * 4];  // dp 0, chunk 0: [stage][cross op] enter, deposited, detected, exit
#define STAT_ADD(i, v) g_cell_stats[(size_t)(blockIdx.x * WARPS + (threadIdx.x >> 5)) * 8 + (i)] += (v)
#else
#define STAT_ADD(i, v)
#endif

struct CellArgs {
  int64_t *rslot;      // [M_cross][Sp] ready slots of small-group memberships
  int64_t *acc;        // [G_large][Sp] max-accumulators of large groups (zeroed per replay)
  int64_t *rres;       // [G_large][Sp] result slots of large groups (parity-encoded like rslot)
  uint32_t *arrive;    // [G_large] arrival counters of large groups (zeroed per replay)
  uint32_t *status;    // [0] = abort flag / error code
  uint64_t timeout_ns;
  int32_t parity;      // ready-slot encoding of this replay: 0 -> t (valid >= 0), 1 -> ~t (valid < 0);
                       // every slot is written once per replay, so the previous replay's values
                       // read as "not yet" and no reset pass is needed
  int32_t n_units;     // cells x chunks of this launch
  int32_t Sp;          // scenario stride (all chunks x 32)
  int32_t chunk0;      // first chunk of this launch
  int32_t nchunks;     // chunks of the whole replay (arrival counters are per chunk)
  uint32_t poll_spin;      // polls before the first sleep
  uint32_t poll_sleep0;    // first sleep (ns), doubled per further poll ...
  uint32_t poll_sleep_max; // ... up to this
  uint32_t fast_spin, fast_sleep0, fast_sleep_max;  // the fast wait's policy (fast_sleep_max 0: off)
  uint32_t lean;       // cross_pairs: 0 off, 1 TP >= 4 cells (default), 2 every cell (PRISM_LEAN, experiments)
  uint32_t mix;        // CTA -> cell permutation stride (1 = identity; odd: a bijection mod a power of two)
  ShardLink L;         // row e: peer exchange buffers (sharded kernels only)
};

// Row e: a cross-shard deposit goes to the copy of every shard holding a member of the group
// (mask bit m = shard m, own shard included); the layout of all copies is identical.
__device__ __forceinline__ int64_t *peer64(const ShardLink &L, int m, int64_t off_bytes) {
  return (int64_t *)(L.base[m] + off_bytes);
}
__device__ __forceinline__ uint32_t *peer32(const ShardLink &L, int m, int64_t off_bytes) {
  return (uint32_t *)(L.base[m] + off_bytes);
}

__device__ __forceinline__ int32_t rank_of(const DevGraph &g, int32_t tp_i, int32_t pp_i, int32_t dp_i) {
  return g.order == PRISM_ORDER_MEGATRON ? tp_i + g.tp * (dp_i + g.dp * pp_i)
                                         : tp_i + g.tp * (pp_i + g.pp * dp_i);
}

// Backoff + watchdog of a waiting warp; returns true when the replay was aborted. The sleep grows
// geometrically from poll_sleep0 to poll_sleep_max ns: a short wait costs one short handoff, a long
// wait (a pipeline stage idling through the 1F1B warm-up) stops stealing issue slots from the
// computing warps of its SM.
__device__ __forceinline__ bool wait_tick(const CellArgs &a, uint32_t &spins, uint64_t &t0, uint32_t sleep0,
                                          uint32_t sleep_max) {
  ++spins;
  if ((threadIdx.x & 31) == 0) STAT_ADD(3, 1);
  const uint32_t sh = min(spins, 16u);
  __nanosleep(min(sleep_max, sleep0 << sh));
  if ((spins & 63) == 0) {
    if (ld_relaxed(a.status) != 0) return true;
    if (t0 == 0) t0 = globaltimer();
    if (globaltimer() - t0 > a.timeout_ns) {
      atomicCAS(a.status, 0u, (uint32_t)PRISM_E_DEADLOCK);
      return true;
    }
  }
  return false;
}

// max over t[0..C) as a balanced tree (depth log2 C instead of a chain of C - 1 dependent maxima)
template <int C>
__device__ __forceinline__ int64_t tree_max(const int64_t (&t)[C]) {
  int64_t m[C];
#pragma unroll
  for (int r = 0; r < C; ++r) m[r] = t[r];
#pragma unroll
  for (int w = 1; w < C; w *= 2)
#pragma unroll
    for (int r = 0; r + w < C; r += 2 * w) m[r] = max(m[r], m[r + w]);
  return m[0];
}

// Sync records of the next cross-cell op, one (rank, slot) pair per lane, loaded right after the
// previous cross op so that their latency overlaps the compute spans in between (the handoff path
// of a rendezvous then starts with no dependent global load).
struct PreRec {
  uint32_t meta, smask;
  int32_t base, grp;
  int64_t dur;
  uint64_t uid;
};

// crec: replica cells, the op's cell record (cell-full ops: one pair, the cell-level group).
template <bool SH>
__device__ __forceinline__ void prefetch_cross(const DevGraph &g, const XOp &xo, const int32_t *rsh, int C,
                                               PreRec &pre, int64_t crec) {
  const int lane = threadIdx.x & 31;
  const int ns = xo.ns;
  if (xo.flags & 1) {
    if (lane == 0) {
      const int32_t h = rsh[0] + xo.hoff;
      pre.meta = g.c_meta[crec];
      pre.base = g.c_base[crec];
      pre.dur = g.h_dur[h];
      pre.uid = g.h_uid[h];
      pre.grp = 0;
      pre.smask = SH ? g.h_smask[h] : 0u;
    }
    return;
  }
  if (ns > 0 && lane < C * ns) {
    const int r = lane / ns, q = lane - r * ns;
    const int32_t h = rsh[r] + xo.hoff + q;
    pre.meta = g.h_meta[h];
    pre.base = g.h_base[h];
    pre.dur = g.h_dur[h];
    pre.uid = g.h_uid[h];
    pre.grp = ns > 1 ? g.node_grp[h] : 0;
    pre.smask = SH ? g.h_smask[h] : 0u;
  }
}

// The exchange arrays a warp polls and accumulates into: the graph's own (unsharded) or its
// shard's exchange buffer (sharded; in a local-group launch the CTA's shard is derived from its
// index), plus the shard index for the lean-path check.
struct XBuf {
  int64_t *rslot, *acc, *rres;
  uint32_t *arrive;
  int32_t self;
};

// Per-warp shared scratch of the cross-cell path.
template <int C>
struct CrossScratch {
  static constexpr int P = C * 4;                      // (rank, slot) pairs: <= 4 slots per op
  static constexpr int L = P * (kSmallGroup - 1);      // poll-list entries
  uint32_t meta[P];   // pair x = r * ns + q: sync record of rank r's q-th group
  int32_t base[P];
  int32_t grp[P];
  int64_t dur[P];
  uint64_t uid[P];
  uint32_t smask[P];  // row e: shards holding members of the pair's group
  int64_t vmax[P][32];  // per pair, per lane: max ready time over the group's members
  // poll list: one entry per (pair, other member) of a small group (ready-slot index) or per large
  // group (arrival-counter index), so a poll round issues every load before folding any of them
  int32_t lidx[L];
  uint8_t lpair[L];   // pair index | 0x80 for a large group's counter
};

// Cross-cell node at template index i for all C ranks of the cell (rare: a few % of ops; kept
// rolled and out of the unrolled per-rank register code so the kernel fits the instruction cache).
// ts[r * 32 + lane] holds rank r's ready time on entry and its finish on exit (shared memory);
// rsh[r] = rank r's first membership slot, hoff = the op's slot offset in the template, ns = slots
// of the op. The op's C x ns sync records are staged in shared memory by one lane-parallel load;
// deposit / arrive for every rank first, then poll (every poll of a pass is an independent load,
// folded on the fly, the own slot is not read back), then finish = max over groups + dur'.
template <bool SH, int C>
__device__ __forceinline__ bool cross_all(const DevGraph &g, const ScenParams &p, const CellArgs &a, const XBuf &xb,
                                          int64_t *__restrict__ gfin, int64_t *ts, int32_t ns,
                                          int32_t k, CrossScratch<C> &cs, const PreRec &pre, int tl, int np) {
  const int lane = threadIdx.x & 31;
  const int32_t Sp = a.Sp;
  const int32_t ck = k / SC;  // np = C * ns pairs (<= 32), or 1 for a replica cell's cell-full op
  if (lane < np) {  // the op's sync records, prefetched into registers one cross op ahead
    cs.meta[lane] = pre.meta;
    cs.base[lane] = pre.base;
    cs.dur[lane] = pre.dur;
    cs.uid[lane] = pre.uid;
    cs.grp[lane] = pre.grp;
    if (SH) cs.smask[lane] = pre.smask;
  }
  __syncwarp();
  bool large_any = false;
  const int64_t pm_dep = a.parity ? -1 : 0;  // slot encoding of this replay
  for (int x = 0, r = 0, q = 0; x < np; ++x) {  // x = r * ns + q, no divisions
    const int64_t tr = ts[r * 32 + lane];
    if (++q == ns) {
      q = 0;
      ++r;
    }
    const uint32_t meta = cs.meta[x];
    const int32_t base = cs.base[x];
    if (!(meta & 0x80000000u)) {
      const int64_t off = (int64_t)(base + (int32_t)((meta >> 16) & 0x7FFF)) * Sp + k;
      const int64_t enc = tr ^ pm_dep;
      if (!SH) {
        st_relaxed64(xb.rslot + off, enc);
      } else {
        for (uint32_t m = cs.smask[x]; m; m &= m - 1)
          st_relaxed_sys64(peer64(a.L, __ffs(m) - 1, a.L.o_rslot) + off, enc);
      }
    } else {
      large_any = true;
      const int64_t off = (int64_t)base * Sp + k;
      if (!SH) {
        red_max(xb.acc + off, tr);
      } else {
        for (uint32_t m = cs.smask[x]; m; m &= m - 1) red_max_sys(peer64(a.L, __ffs(m) - 1, a.L.o_acc) + off, tr);
      }
    }
  }
  uint32_t large_done = 0;  // !SH: large pairs this warp completed as their last arriver
  if (large_any) {
    if (SH) {
      // the accumulations are performed before the arrival is counted (system scope: peers)
      __threadfence_system();
      __syncwarp();
      if (lane == 0)
        for (int x = 0; x < np; ++x)
          if (cs.meta[x] & 0x80000000u) {
            const int64_t ai = (int64_t)cs.base[x] * a.nchunks + ck;
            for (uint32_t m = cs.smask[x]; m; m &= m - 1)
              atomicAdd_system(peer32(a.L, __ffs(m) - 1, a.L.o_arrive) + ai, 1u);
          }
    } else {
      // last arriver publishes: the lanes' red.max are ordered before lane 0's acq_rel arrival
      // (bar.warp.sync orders the warp's memory operations); the member whose arrival completes
      // the count reads the accumulator (acquire: every member's max is visible) and writes the
      // group's max into a value-as-flag result slot, which the other members poll like a
      // ready slot — no fence on anyone's path
      __syncwarp();
      if (lane == 0)
        for (int x = 0; x < np; ++x)
          if (cs.meta[x] & 0x80000000u) {
            const int64_t ai = (int64_t)cs.base[x] * a.nchunks + ck;
            uint32_t old;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(xb.arrive + ai) : "memory");
            if (old + 1 == (cs.meta[x] & 0xFFFF)) large_done |= 1u << x;
          }
      large_done = __shfl_sync(0xffffffffu, large_done, 0);
      __syncwarp();
      for (uint32_t m = large_done; m; m &= m - 1) {
        const int x = __ffs(m) - 1;
        const int64_t off = (int64_t)cs.base[x] * Sp + k;
        const int64_t v = ld_relaxed64(xb.acc + off);
        st_relaxed64(xb.rres + off, v ^ pm_dep);
        cs.vmax[x][lane] = v;
      }
    }
  }
#ifdef PRISM_CELL_STATS
  if (tl >= 0 && lane == 0) g_tl[tl * 4 + 1] = globaltimer();
#endif
  // poll until every (rank, group) pair of the op is resolved. The (pair, member) loads of a
  // round are flattened into one list and issued kPollBatch at a time before any is folded (a loop with a
  // load-dependent branch per pair would serialise one L2 round trip per pair); a pair resolved
  // for this lane is not polled again. Slot values are parity-encoded: v ^ pm is the ready time
  // when >= 0; a large group is resolved when its arrival counter reaches its size.
  const int64_t pm = a.parity ? -1 : 0;
  int32_t nl;
  {
    int32_t cnt = 0;
    uint32_t meta = 0;
    if (lane < np) {
      meta = cs.meta[lane];
      cnt = (meta & 0x80000000u) ? 1 : (int32_t)(meta & 0xFFFF) - 1;
    }
    int32_t incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    nl = __shfl_sync(0xffffffffu, incl, 31);
    if (lane < np) {
      int32_t o = incl - cnt;
      const int32_t base = cs.base[lane];
      if (meta & 0x80000000u) {
        cs.lidx[o] = base;
        cs.lpair[o] = (uint8_t)(lane | 0x80);
      } else {
        const int32_t size = (int32_t)(meta & 0xFFFF), own = (int32_t)((meta >> 16) & 0x7FFF);
        for (int32_t mm = 0; mm < size; ++mm)
          if (mm != own) {
            cs.lidx[o] = base + mm;
            cs.lpair[o] = (uint8_t)lane;
            ++o;
          }
      }
    }
    for (int r = 0, x = 0; r < C; ++r) {
      const int64_t tr = ts[r * 32 + lane];
      for (int q = 0; q < ns; ++q, ++x)
        if (!((large_done >> x) & 1u)) cs.vmax[x][lane] = tr;  // completed large pairs hold the max
    }
    __syncwarp();
  }
  uint32_t pending = (np >= 32 ? 0xFFFFFFFFu : ((1u << np) - 1u)) & ~large_done;
  uint32_t spins = 0;
  uint64_t tw = 0;
  // fast wait: spin on ONE pending entry — the last of the list, which the partners deposit last
  // (they deposit rank by rank in the same order) — with a loop of a few instructions, so a long
  // wait costs its SM almost no issue slots and the handoff is detected within one short sleep;
  // the full rounds below then usually resolve everything at once
  if (a.fast_sleep_max) {
    int32_t jr = nl - 1;
    while (jr >= 0 && !((pending >> (cs.lpair[jr] & 31)) & 1u)) --jr;
    if (jr >= 0) {
      const uint32_t pr = cs.lpair[jr];
      const int32_t idx = cs.lidx[jr];
      const bool cnt = (pr & 0x80) && SH;
      const int64_t *p64 = (pr & 0x80) ? xb.rres + (int64_t)idx * Sp + k : xb.rslot + (int64_t)idx * Sp + k;
      const uint32_t *p32 = xb.arrive + (int64_t)idx * a.nchunks + ck;
      const int64_t need = (int64_t)(cs.meta[pr & 31] & 0xFFFF);
      uint32_t fs = 0, fsl = 0;
      while (true) {
        const int64_t v = cnt ? (int64_t)poll32<SH>(p32) - need : poll64<SH>(p64) ^ pm;
        if (__all_sync(0xffffffffu, v >= 0)) break;
        if (fs < a.fast_spin) ++fs;
        else if (wait_tick(a, fsl, tw, a.fast_sleep0, a.fast_sleep_max)) return false;
      }
    }
  }
  while (true) {
    uint32_t bad = 0;
    for (int32_t j0 = 0; j0 < nl; j0 += kPollBatch) {
      int64_t v[kPollBatch];
#pragma unroll
      for (int u = 0; u < kPollBatch; ++u) {
        const int32_t j = j0 + u;
        v[u] = 0;
        if (j < nl) {
          const uint32_t pr = cs.lpair[j];
          if ((pending >> (pr & 31)) & 1u) {
            const int32_t idx = cs.lidx[j];
            if ((pr & 0x80) && SH)
              v[u] = (int64_t)poll32<SH>(xb.arrive + (int64_t)idx * a.nchunks + ck) -
                     (int64_t)(cs.meta[pr & 31] & 0xFFFF);
            else if (pr & 0x80)  // the large group's result slot (published by its last arriver)
              v[u] = poll64<SH>(xb.rres + (int64_t)idx * Sp + k) ^ pm;
            else
              v[u] = poll64<SH>(xb.rslot + (int64_t)idx * Sp + k) ^ pm;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kPollBatch; ++u) {
        const int32_t j = j0 + u;
        if (j < nl) {
          const uint32_t pr = cs.lpair[j];
          const int x = pr & 31;
          if ((pending >> x) & 1u) {
            if (v[u] < 0) bad |= 1u << x;
            else if (!(pr & 0x80) || !SH) cs.vmax[x][lane] = max(cs.vmax[x][lane], v[u]);
          }
        }
      }
    }
    pending &= bad;
    if (__all_sync(0xffffffffu, pending == 0)) break;
    if (++spins > a.poll_spin && wait_tick(a, spins, tw, a.poll_sleep0, a.poll_sleep_max)) return false;
  }
#ifdef PRISM_CELL_STATS
  if (tl >= 0 && lane == 0) g_tl[tl * 4 + 2] = globaltimer();
#endif
  if (large_any && SH) fence_acq_rel_sys();
  for (int r = 0; r < C && r * ns < np; ++r) {
    int64_t fr = 0;
    for (int32_t q = 0; q < ns; ++q) {
      const int x = r * ns + q;
      int64_t m = ((cs.meta[x] & 0x80000000u) && SH) ? __ldcg(xb.acc + (int64_t)cs.base[x] * Sp + k) : cs.vmax[x][lane];
      const int64_t gd = cs.dur[x];
      const uint64_t uid = cs.uid[x];
      const uint32_t gb = (uid >> 56) == PRISM_ROLE_P2P ? 4u : 2u;
      const int32_t kg = p.first + k;  // global scenario index (perturbation key)
      if ((p.mask & gb) && p.amp > 0 && kg > 0) m += perturb_x(gd, p.seed ^ ((uint64_t)kg * K_GOLD) ^ (uid * K_MIX), p);
      else m += gd;
      fr = max(fr, m);
      if (ns > 1) gfin[(int64_t)cs.grp[x] * Sp + k] = m;  // P2P-batch group finishes, for queries
    }
    ts[r * 32 + lane] = fr;
  }
  __syncwarp();
  return true;
}

// Lean cross-cell path for the common op whose every (rank, slot) pair is a 2-member small group
// (a P2P message, reading Z3, or a 2-member EDP group) on an unsharded replay: lane x < C * ns
// holds pair x's prefetched record, so its own and its partner's ready-slot indices come by
// shuffle — no record staging, no poll list — and a poll round is one independent load per pending
// pair, issued kPollBatch at a time before any is folded. Same slots, encoding and results as
// cross_all (which handles every other op).
template <int C>
__device__ __forceinline__ bool cross_pairs(const ScenParams &p, const CellArgs &a, const XBuf &xb, int64_t *__restrict__ gfin,
                                            int64_t *ts, int32_t ns, int32_t k, CrossScratch<C> &cs,
                                            const PreRec &pre, int tl) {
  const int lane = threadIdx.x & 31;
  const int32_t Sp = a.Sp;
  const int np = C * ns;  // <= 32
  constexpr int PB = C <= 2 ? 4 : kPollBatch;  // loads per batch (small cells: fewer live registers)
  const int64_t pm = a.parity ? -1 : 0;  // slot encoding of this replay
  const int32_t own = (int32_t)((pre.meta >> 16) & 0x7FFF);
  const int32_t oslot = pre.base + own, pslot = pre.base + (own ^ 1);
  for (int x = 0, r = 0, q = 0; x < np; ++x) {  // deposit every pair first: no self-wait
    const int32_t os = __shfl_sync(0xffffffffu, oslot, x);
    st_relaxed64(xb.rslot + (int64_t)os * Sp + k, ts[r * 32 + lane] ^ pm);
    if (++q == ns) {
      q = 0;
      ++r;
    }
  }
#ifdef PRISM_CELL_STATS
  if (tl >= 0 && lane == 0) g_tl[tl * 4 + 1] = globaltimer();
#endif
  uint32_t pending = np >= 32 ? 0xFFFFFFFFu : ((1u << np) - 1u);
  uint32_t spins = 0, fs = 0, fsl = 0;
  uint64_t tw = 0;
  const int32_t kg = p.first + k;  // global scenario index (perturbation key)
  const bool pert_ok = p.amp > 0 && kg > 0;
  const uint64_t sx = p.seed ^ ((uint64_t)kg * K_GOLD);
  if (a.fast_sleep_max) {  // fast wait on the pair the partners deposit last (see cross_all)
    const int32_t ps = __shfl_sync(0xffffffffu, pslot, np - 1);
    const int64_t *p64 = xb.rslot + (int64_t)ps * Sp + k;
    while (!__all_sync(0xffffffffu, (ld_relaxed64(p64) ^ pm) >= 0)) {
      if (fs < a.fast_spin) ++fs;
      else if (wait_tick(a, fsl, tw, a.fast_sleep0, a.fast_sleep_max)) return false;
    }
  }
  while (true) {
    for (int x0 = 0; x0 < np; x0 += PB) {
      int64_t v[PB];
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        const int x = x0 + u;
        const int32_t ps = __shfl_sync(0xffffffffu, pslot, x & 31);
        v[u] = -1;
        if (x < np && ((pending >> x) & 1u)) v[u] = ld_relaxed64(xb.rslot + (int64_t)ps * Sp + k) ^ pm;
      }
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        const int x = x0 + u;
        if (x < np && ((pending >> x) & 1u) && v[u] >= 0) {
          cs.vmax[x][lane] = v[u];
          pending &= ~(1u << x);
        }
      }
    }
    if (__all_sync(0xffffffffu, pending == 0)) break;
    if (++spins > a.poll_spin && wait_tick(a, spins, tw, a.poll_sleep0, a.poll_sleep_max)) return false;
  }
#ifdef PRISM_CELL_STATS
  if (tl >= 0 && lane == 0) g_tl[tl * 4 + 2] = globaltimer();
#endif
  // finish = max(own, partner) + dur'_g; one slot per rank (the common case): unrolled over the
  // ranks so the C hashes run as independent chains
  if (ns == 1) {  // the pairs of one op share a role (all P2P messages, or all EDP groups)
    int64_t tt[C], dd[C];
    uint64_t xx[C];
#pragma unroll
    for (int r = 0; r < C; ++r) {
      dd[r] = __shfl_sync(0xffffffffu, pre.dur, r);
      const uint64_t uid = __shfl_sync(0xffffffffu, pre.uid, r);
      xx[r] = sx ^ (uid * K_MIX);
      tt[r] = max(ts[r * 32 + lane], cs.vmax[r][lane]);
    }
    const uint32_t gb = (__shfl_sync(0xffffffffu, pre.uid, 0) >> 56) == PRISM_ROLE_P2P ? 4u : 2u;
    if ((p.mask & gb) && pert_ok) {
      perturb_add<C>(tt, dd, xx, p);
    } else {
#pragma unroll
      for (int r = 0; r < C; ++r) tt[r] += dd[r];
    }
#pragma unroll
    for (int r = 0; r < C; ++r) ts[r * 32 + lane] = tt[r];
  } else {
    for (int r = 0, x = 0; r < C; ++r) {
      const int64_t tr = ts[r * 32 + lane];
      int64_t fr = 0;
      for (int32_t q = 0; q < ns; ++q, ++x) {
        const int64_t gd = __shfl_sync(0xffffffffu, pre.dur, x);
        const uint64_t uid = __shfl_sync(0xffffffffu, pre.uid, x);
        const int32_t grp = __shfl_sync(0xffffffffu, pre.grp, x);
        const uint32_t gb = (uid >> 56) == PRISM_ROLE_P2P ? 4u : 2u;
        const int64_t m = max(tr, cs.vmax[x][lane]) + (((p.mask & gb) && pert_ok) ? perturb_x(gd, sx ^ (uid * K_MIX), p) : gd);
        fr = max(fr, m);
        gfin[(int64_t)grp * Sp + k] = m;  // P2P-batch group finishes, for queries
      }
      ts[r * 32 + lane] = fr;
    }
  }
  __syncwarp();
  return true;
}

// Dynamic shared memory of one warp of an EP CTA: cross scratch, chain state, membership slots.
template <int C>
__host__ __device__ constexpr size_t cta_warp_scratch() {
  return (sizeof(CrossScratch<C>) + C * 32 * 8 + MAX_TP * 4 + 15) / 16 * 16;
}

// PR (rows f1/f3/f4): the graph carries per-node durations (prism_set_durations), so a compute
// span or chained collective lasts its own rank's value node_sdur[rb[r] + i], loaded one op ahead.
// MS (row f2, multi-stream ranks): besides its ranks' ready times the warp keeps, per rank, the
// finish of the last op of each stream and the latest record of each (densely renumbered) event
// slot in dynamic shared memory; an op starts at max(its stream's last finish, its awaited
// event). The ranks of a cell still share one template, so TP collectives stay register-local.
// KS > 1 (EP CTAs, replica cells): the KS cells of one EP group are the KS warps of one CTA; an
// EP collective (class 4) is the max over the CTA's ranks, formed in registers and shared memory
// behind one CTA barrier. A warp of such a CTA never leaves the loop early (after an abort it
// skips the remaining waits), so the CTA's barrier counts always match.
template <int C, bool SH, bool PR, bool MS, int KS = 1>
__global__ void __launch_bounds__(KS * 32, KS > 8 ? 1 : (KS > 1 ? 2 : (C == 1 ? 28 : (C == 2 ? 24 : 16)))) cell_kernel(DevGraph g, ScenParams p, CellArgs a,
                                                         int64_t *__restrict__ fin,
                                                         int64_t *__restrict__ gfin,
                                                         int64_t *__restrict__ rank_end) {
  const int lane = threadIdx.x & 31;
  const int sub = KS > 1 ? (int)(threadIdx.x >> 5) : 0;  // the warp's cell within the CTA
  const int32_t unit = blockIdx.x;                        // CTA (KS cells)
  if (unit >= a.n_units) return;  // the whole CTA
  bool aborted = unit == g.stall_unit;  // stall_unit: watchdog test hook (no arrivals at all)
  if (KS == 1 && aborted) return;
  constexpr bool PAIR = C >= 4 && !PR && !MS;  // (compute, TP) pairs in one iteration
  // row e: this CTA's shard (a local-group launch covers every shard of the device, units grouped
  // by shard) and its DP block, exchange buffer and output arrays
  int32_t shard = SH ? a.L.self : 0, d0 = g.d0, d1 = g.d1, s0 = g.s0, s1 = g.s1, u = unit;
  int64_t fnode0 = g.fin_node0;
  if (SH && a.L.lg > 0) {
    const int32_t per = a.n_units / a.L.lg;
    shard = unit / per;
    u = unit - shard * per;
    if (g.shard_axis == 1) {  // PP-stage blocks: every shard keeps all rows
      const int32_t blk = g.pp / g.n_shards;
      s0 = shard * blk;
      s1 = s0 + blk;
    } else {
      const int32_t blk = g.dp / g.n_shards;
      d0 = shard * blk;
      d1 = d0 + blk;
      // a DP block is one contiguous row range under TP_PP_DP; Megatron order keeps all rows
      fnode0 = g.order == PRISM_ORDER_MEGATRON ? 0 : (int64_t)shard * g.fin_rows;
    }
    fin = a.L.lg_fin[shard];
    gfin = a.L.lg_gfin[shard];
    rank_end = a.L.lg_rank_end[shard];
  }
  XBuf xb{a.rslot, a.acc, a.rres, a.arrive, shard};
  if (SH) {
    unsigned char *eb = a.L.base[shard];
    xb.rslot = (int64_t *)(eb + a.L.o_rslot);
    xb.acc = (int64_t *)(eb + a.L.o_acc);
    xb.rres = nullptr;
    xb.arrive = (uint32_t *)(eb + a.L.o_arrive);
  }
  const int32_t nst = s1 - s0;
  const int32_t RC = g.cell_R > 1 ? g.cell_R : 1;  // replica cells: RC = C consecutive DP replicas
  const int32_t cells = nst * (d1 - d0) / RC / KS;  // this shard's CTAs of one chunk
  const int32_t cell = (int32_t)(((uint64_t)(u % cells) * a.mix) % (uint64_t)cells), chunk = a.chunk0 + u / cells;
  const int32_t s = s0 + cell % nst, dpi = d0 + ((cell / nst) * KS + sub) * RC;
  // rank r of the cell: tp index r (TP cells) or DP replica dpi + r (replica cells, tp = 1)
  auto cell_rank = [&](int32_t r) { return RC > 1 ? rank_of(g, 0, s, dpi + r) : rank_of(g, r, s, dpi); };
  const int64_t crec0 = RC > 1 ? g.crec_ptr[s] + (int64_t)(dpi / RC) * (g.x_ptr[s + 1] - g.x_ptr[s]) - g.x_ptr[s] : 0;
  const int32_t Sp = a.Sp;
  const int32_t k = chunk * SC + lane;
  // per-warp scratch: static for one warp per CTA, carved from dynamic shared memory for EP CTAs
  // (KS warps' scratch exceeds the 48 KB of static shared memory)
  __shared__ int64_t ts_s[KS == 1 ? C * 32 : 1];  // chain state of the cross-cell path
  __shared__ CrossScratch<KS == 1 ? C : 1> cs_s;
  __shared__ int32_t rsh_s[KS == 1 ? MAX_TP : 1];  // first membership slot of each rank
  extern __shared__ __align__(16) unsigned char dsm[];
  int64_t *ts;
  CrossScratch<C> *csp;
  int32_t *rsh;
  int64_t *xm = nullptr;  // EP CTAs: [2][KS][32] partial maxima (double-buffered)
  size_t dyn_used = 0;
  if (KS == 1) {
    ts = ts_s;
    csp = reinterpret_cast<CrossScratch<C> *>(&cs_s);
    rsh = rsh_s;
  } else {
    const size_t per = cta_warp_scratch<C>();
    unsigned char *w = dsm + (size_t)sub * per;
    csp = reinterpret_cast<CrossScratch<C> *>(w);
    ts = reinterpret_cast<int64_t *>(w + sizeof(CrossScratch<C>));
    rsh = reinterpret_cast<int32_t *>(w + sizeof(CrossScratch<C>) + C * 32 * 8);
    xm = reinterpret_cast<int64_t *>(dsm + (size_t)KS * per);
    dyn_used = (size_t)KS * per + 2 * KS * 32 * 8;
  }
  CrossScratch<C> &cs = *csp;
  int xp = 0;
  int32_t rb[C];
  int32_t rs[C];   // first membership slot of each rank (node_gptr of its first node)
  uint32_t rkh[C];  // high word of (rank << 32) * K_MIX (its low word is zero): a compute span's
                    // uid mix is that + tidx * K_MIX (perturb_add_span)
#pragma unroll
  for (int r = 0; r < C; ++r) {
    const int32_t rr = cell_rank(r);
    rb[r] = g.rank_ptr[rr];
    rs[r] = g.node_gptr[rb[r]];
    rkh[r] = (uint32_t)((((uint64_t)rr << 32) * K_MIX) >> 32);
    if (lane == 0) rsh[r] = rs[r];
  }
  __syncwarp();
  const int32_t len = g.rank_ptr[cell_rank(0) + 1] - rb[0];
  const int32_t kg = p.first + k;  // global scenario index (perturbation key)
  const uint64_t sx = p.seed ^ ((uint64_t)kg * K_GOLD);
  // per-warp flags pinned in a register (an asm output cannot be rematerialised from the kernel
  // parameters, which the compiler otherwise reloads on every op)
  uint32_t fl = (((p.mask & 1u) && p.amp > 0 && kg > 0) ? 1u : 0u) | (((p.mask & 2u) && p.amp > 0 && kg > 0) ? 2u : 0u) |
                (p.record ? 4u : 0u);
  asm volatile("" : "+r"(fl));
  const bool cpert = fl & 1u, gpert = fl & 2u, record = fl & 4u;
  int64_t t[C];
#pragma unroll
  for (int r = 0; r < C; ++r) t[r] = 0;
  // MS state: [stream][rank][lane] then [event][rank][lane] (g.ms_streams, g.ms_events)
  int64_t *ms_dyn = reinterpret_cast<int64_t *>(dsm + dyn_used) +
                    (KS > 1 ? (size_t)sub * (g.ms_streams + g.ms_events) * C * 32 : 0);
  if (MS) {
    for (int x = 0; x < (g.ms_streams + g.ms_events) * C; ++x) ms_dyn[x * 32 + lane] = 0;  // unrecorded: satisfied
  }
#ifdef PRISM_CELL_STATS
  const long long k_start = clock64();
  if (lane == 0) STAT_ADD(4, globaltimer());
#endif
  // cross-op cursor of the stage template and the prefetched records of the next cross op
  int32_t xk = g.x_ptr[s];
  const int32_t xend = g.x_ptr[s + 1];
  XOp xo{len, 0, 0, 0};
  PreRec pre{0u, 0u, 0, 0, 0, 0};
  if (xk < xend) {
    xo = g.x_ops[xk];
    prefetch_cross<SH>(g, xo, rsh, C, pre, crec0 + xk);
  }
  // the XOp entry of the cross op after next, loaded a cross op early: prefetching the next op's
  // records right after a cross op then does not first wait for its entry
  XOp xq{len, 0, 0, 0};
  if (xk + 1 < xend) xq = g.x_ops[xk + 1];
  int64_t pd[PR ? C : 1];  // PR: per-rank durations of the next op
  if (PR) {
#pragma unroll
    for (int r = 0; r < C; ++r) pd[r] = len > 0 ? __ldg(g.node_sdur + rb[r]) : 0;
  }
  // op records of the stage template (the cell's ranks share it; the per-rank part of a compute
  // span's uid is rkh[r]): class, record duration (PR: the rank-0 node's override, e.g. a group's
  // max over its members' overridden durations) and, for in-cell / chained / CTA-local group ops,
  // the uid of the cell's rank-0 group (closed form from the template's packed group word),
  // 32 ops per coalesced round trip from the L2-resident tables, next batch in flight
  const int64_t top0 = g.t_op0[s];
  const int32_t tp0 = 0, dp0 = dpi;  // coordinates of the cell's rank 0
  auto load_rec = [&](int32_t i, uint32_t &cls, int64_t &d, uint64_t &ux, uint32_t &msv) {
    const int64_t op = top0 + i;
    cls = __ldg(g.t_cls + op);
    d = PR ? __ldg(g.node_sdur + rb[0] + i) : __ldg(g.t_sdur + op);
    ux = 0;
    if ((cls & 0xFu) != 0 && (cls & 0xFu) != 2) {
      const uint64_t qi = __ldg(g.t_qinfo + op);
      ux = group_uid_packed(g, qi, group_inst(g, (int32_t)(qi & 0xFF), tp0, dp0, dp0 % g.ep, dp0 / g.ep));
    }
    if (MS) msv = __ldg(g.t_ms + op);
  };
  uint32_t ncls = 2, nms = 0;
  int64_t nd = 0;
  uint64_t nux = 0;
  if (lane < len) load_rec(lane, ncls, nd, nux, nms);
  // fin rows of op i (graph.h fin_off): the cell's C ranks are C consecutive 32-lane rows of this
  // chunk, and op i + 1's rows follow: one moving pointer, rank r at the constant offset r * 32
  int64_t *fp = fin ? fin + (((int64_t)(k / SC) * g.fin_rows + cell_row0(g, cell_rank(0)) - fnode0) * SC + (k % SC))
                    : nullptr;
  for (int32_t base = 0; base < len; base += 32) {
    const int32_t cnt = min(32, len - base);
    const uint32_t bcls = ncls;
    const int64_t bd = nd;
    const uint64_t bux = nux;
    const uint32_t bms = nms;
    if (base + 32 + lane < len) load_rec(base + 32 + lane, ncls, nd, nux, nms);
    // op j's class / duration were fetched during op j-1 (software pipelined: the dispatch
    // branch of an op does not wait on its shuffles)
    uint32_t c_n = __shfl_sync(0xffffffffu, bcls, 0);
    int64_t d_n = __shfl_sync(0xffffffffu, bd, 0);
    for (int32_t j = 0; j < cnt; ++j) {
      const uint32_t c = c_n & 0xFu;
      const uint32_t cfl = c_n;  // class flags (0x10 pair, 0x20 / 0x40 replica-cell uid steps)
      // pair: this compute span is followed by a TP collective of this batch (plan flag 0x10);
      // both run in this iteration (plain variant only)
      const bool pair = PAIR && (c_n & 0x10u) && j + 1 < cnt;
      const int64_t d = d_n;
      const int32_t i = base + j;
      c_n = __shfl_sync(0xffffffffu, bcls, (j + 1) & 31);
      d_n = __shfl_sync(0xffffffffu, bd, (j + 1) & 31);
      int64_t *ms_sp = nullptr, *ms_rp = nullptr;  // MS: this op's stream / recorded-event rows
      if (MS) {  // row f2: the op's stream / event edges (same for every rank of the cell)
        const uint32_t mb = __shfl_sync(0xffffffffu, bms, j);
        const uint32_t st = mb & 15u, rec = (mb >> 4) & 15u, wt = (mb >> 8) & 15u;
        ms_sp = ms_dyn + st * C * 32 + lane;
        ms_rp = rec ? ms_dyn + (g.ms_streams + rec - 1) * C * 32 + lane : nullptr;
        const int64_t *wp = wt ? ms_dyn + (g.ms_streams + wt - 1) * C * 32 + lane : nullptr;
#pragma unroll
        for (int r = 0; r < C; ++r) {
          int64_t rd = ms_sp[r * 32];
          if (wp) rd = max(rd, wp[r * 32]);
          t[r] = rd;
        }
      }
      int64_t dr[PR ? C : 1];  // PR: this op's per-rank durations (loaded during the previous op)
      if (PR) {
#pragma unroll
        for (int r = 0; r < C; ++r) {
          dr[r] = pd[r];
          if (i + 1 < len) pd[r] = __ldg(g.node_sdur + rb[r] + i + 1);
        }
      }
      if (pair) {  // compute span i, then the TP collective i + 1 (its hash beside the span chains)
        const uint64_t uxn = __shfl_sync(0xffffffffu, bux, (j + 1) & 31);
        int64_t tq = d_n;
        if (cpert) {  // the TP hash as a ninth chain beside the span's
          tq = perturb_add_span_q<C>(t, d, sx, rkh, (uint64_t)i * K_MIX, d_n, sx ^ (uxn * K_MIX), gpert, p);
        } else {
          if (gpert) tq = perturb_x(d_n, sx ^ (uxn * K_MIX), p);
#pragma unroll
          for (int r = 0; r < C; ++r) t[r] += d;
        }
        if (record) {  // op i's finishes; the tail below writes op i + 1's
#pragma unroll
          for (int r = 0; r < C; ++r) __stcs(fp + r * SC, (long long)t[r]);
          fp += C * SC;
        }
        const int64_t m = tree_max<C>(t) + tq;
#pragma unroll
        for (int r = 0; r < C; ++r) t[r] = m;
        ++j;  // op i + 1 done
        c_n = __shfl_sync(0xffffffffu, bcls, (j + 1) & 31);
        d_n = __shfl_sync(0xffffffffu, bd, (j + 1) & 31);
      } else if (c == 0) {  // compute span: every rank waits out its own perturbed duration
        if (cpert) {
          int64_t dd[C];
#pragma unroll
          for (int r = 0; r < C; ++r) dd[r] = PR ? dr[r] : d;
          perturb_add_span<C, PR>(t, dd, sx, rkh, (uint64_t)i * K_MIX, p);
        } else {
#pragma unroll
          for (int r = 0; r < C; ++r) t[r] += PR ? dr[r] : d;
        }
      } else if (KS > 1 && c == 4) {  // EP collective of an EP CTA: the group is this CTA's ranks
        const uint64_t ux = __shfl_sync(0xffffffffu, bux, j);
        int64_t m = tree_max<C>(t);
        xm[(xp * KS + sub) * 32 + lane] = m;
        __syncthreads();
#pragma unroll
        for (int w = 0; w < KS; ++w) m = max(m, xm[(xp * KS + w) * 32 + lane]);
        xp ^= 1;
        m += gpert ? perturb_x(d, sx ^ (ux * K_MIX), p) : d;
#pragma unroll
        for (int r = 0; r < C; ++r) t[r] = m;
      } else if (c == 1) {  // in-cell TP collective: register-local segmented max
        const uint64_t ux = __shfl_sync(0xffffffffu, bux, j);
        int64_t m = tree_max<C>(t);
        m += gpert ? perturb_x(d, sx ^ (ux * K_MIX), p) : d;
#pragma unroll
        for (int r = 0; r < C; ++r) t[r] = m;
      } else if (c == 3) {  // chained collective: every member is ready at the previous
                            // occurrence's shared finish, so start = own ready time (exact)
        const uint64_t ux = __shfl_sync(0xffffffffu, bux, j);
        if (gpert) {
          // rank r's group uid = ux + r * 2^24 (gid = tp_i + ...), WORLD: one group; replica cells:
          // a per-replica group (flag 0x20, gid = s + pp * dp) steps by pp, a cell-full one (0x40)
          // is one group for the whole cell
          const uint64_t um = ux * K_MIX;
          const uint32_t cf = cfl;
          const uint64_t step = (cf & 0x40u) ? 0ull
                                : (cf & 0x20u) ? ((uint64_t)g.pp << 24)
                                : ((ux >> 56) == PRISM_ROLE_WORLD ? 0ull : (1ull << 24));
          const uint64_t stepm = step * K_MIX;
          int64_t dd[C];
          uint64_t xx[C];
#pragma unroll
          for (int r = 0; r < C; ++r) {
            dd[r] = PR ? dr[r] : d;
            xx[r] = sx ^ (um + (uint64_t)r * stepm);
          }
          perturb_add<C>(t, dd, xx, p);
        } else {
#pragma unroll
          for (int r = 0; r < C; ++r) t[r] += PR ? dr[r] : d;
        }
      } else {  // cross-cell synchronization, rank by rank (deposit all first: no self-wait)
#ifdef PRISM_CELL_STATS
        const long long c0 = clock64();
#endif
        int tl = -1;
#ifdef PRISM_CELL_STATS
        if (k < 32 && dpi == 0 && s < 16 && xk - g.x_ptr[s] < 128) tl = s * 128 + (xk - g.x_ptr[s]);
        if (tl >= 0 && lane == 0) g_tl[tl * 4 + 0] = globaltimer();
#endif
        // replica cells, cell-full group (DP / EP / WORLD over the cell's replicas): the cell's
        // members reach it together, so the warp enters with their max as ONE member (pair 0)
        const bool cfull = xo.flags & 1;
        if (cfull) {
          const int64_t m = tree_max<C>(t);
#pragma unroll
          for (int r = 0; r < C; ++r) t[r] = m;
        }
#pragma unroll
        for (int r = 0; r < C; ++r) ts[r * 32 + lane] = t[r];
        __syncwarp();
        // every pair a 2-member small group (P2P messages): the lean path (TP >= 4 cells; for
        // TP = 1 / 2 cells it measured slower than cross_all on C4). Sharded: only groups whose
        // members are all on this shard (P2P messages never leave a DP block, reading R9) — no
        // peer touches their ready slots in the local exchange buffer, so gpu scope suffices
        const bool lean = !cfull && (C >= 4 || a.lean > 1) && a.lean &&
                          __all_sync(0xffffffffu, lane >= C * xo.ns || ((pre.meta & 0x8000FFFFu) == 2u &&
                                                                        (!SH || pre.smask == (1u << xb.self))));
        // after an abort (watchdog, or the stall test hook) no more arrivals or waits: the warp
        // runs to the end (EP CTAs keep their barriers matched), its results are invalid
        const bool ok = aborted ? false
                        : lean  ? cross_pairs<C>(p, a, xb, gfin, ts, xo.ns, k, cs, pre, tl)
                                : cross_all<SH, C>(g, p, a, xb, gfin, ts, xo.ns, k, cs, pre, tl, cfull ? 1 : C * xo.ns);
        __syncwarp();
#pragma unroll
        for (int r = 0; r < C; ++r) t[r] = ts[(cfull ? 0 : r) * 32 + lane];
#ifdef PRISM_CELL_STATS
        if (tl >= 0 && lane == 0) g_tl[tl * 4 + 3] = globaltimer();
#endif
        if (!ok) {
          if (KS == 1) return;
          aborted = true;
        }
        if (++xk < xend) {  // next cross op: its records load while the compute spans run
          xo = xq;
          prefetch_cross<SH>(g, xo, rsh, C, pre, crec0 + xk);
          if (xk + 1 < xend) xq = g.x_ops[xk + 1];
        }
#ifdef PRISM_CELL_STATS
        if (lane == 0) {
          const long long dc = clock64() - c0;
          STAT_ADD(1, dc);
          if (s < 16 && i < 4096) atomicAdd(&g_wait_hist[s * 4096 + i], (unsigned long long)dc);
        }
#endif
      }
      if (MS) {
#pragma unroll
        for (int r = 0; r < C; ++r) {
          ms_sp[r * 32] = t[r];
          if (ms_rp) ms_rp[r * 32] = t[r];
        }
      }
      if (record) {
#pragma unroll
        for (int r = 0; r < C; ++r) {
          __stcs(fp + r * SC, (long long)t[r]);
        }
        fp += C * SC;
      }
    }
  }
  if (MS) {  // a multi-stream rank ends with its last stream
#pragma unroll
    for (int r = 0; r < C; ++r)
      for (int x = 0; x < g.ms_streams; ++x) t[r] = max(t[r], ms_dyn[(x * C + r) * 32 + lane]);
  }
#pragma unroll
  for (int r = 0; r < C; ++r) rank_end[(int64_t)cell_rank(r) * Sp + k] = t[r];
#ifdef PRISM_CELL_STATS
  if (lane == 0) {
    STAT_ADD(0, clock64() - k_start);
    STAT_ADD(5, globaltimer());
  }
#endif
}

}  // namespace

// type-erased kernel pointer of one variant (cells_k_*.cu): tp = cell width (tp, or the replicas
// of a replica cell), ks = warps (cells) per CTA: 1, or 8 / 16 for EP CTAs (width 2, 4 or 8 / 2 or 4)
const void *cell_kernel_get(int tp, bool sh, bool pr, bool ms, int ks);

}  // namespace prism
