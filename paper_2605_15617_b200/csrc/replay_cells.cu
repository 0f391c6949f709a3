// replay_cells.cu — the cell kernel: one persistent cooperative launch replays every rank (rows
// a6-a8).
//
// Same semantics as replay.cu (readings Z2-Z5), different
// schedule. A *cell* is one TP group: the tp ranks of a (stage, dp) pair. They run the same stage
// template, so they walk it in lockstep, and every TP collective's members are exactly the
// cell. One warp owns one (cell, 32-scenario chunk): lane = scenario, and the lane keeps the chain
// state t[r] of all tp ranks of the cell in registers. Per template op:
//   compute span      : t[r] += dur'(rank r)            tp independent hash chains per lane (ILP)
//   TP collective     : t[r] = max_r t[r] + dur'_g      the segmented max is register-local
//   small cross-cell  : (P2P message, EP/EDP groups of <= 8) every member stores its ready time into
//   group               its global ready slot and polls the other members' slots until they are
//                       valid: an aligned 8-byte store is single-copy atomic, so the value is its own
//                       flag (parity-encoded per replay, see CellArgs) and no fence is needed
//   large cross-cell  : (DP, WORLD, big EP) red.max of the ready times into the group's accumulator,
//   group               then one acq_rel arrival per warp on its counter; the member completing the
//                       count reads the accumulator and publishes the maximum in a value-as-flag
//                       result slot the others poll (sharded replays: fenced system-scope variant,
//                       members poll the counter, then read the accumulator)
// and a node finishes at the max over its groups' (start + dur'_g) (reading Z3). Ops whose pairs
// are all 2-member groups take the lean path (cross_pairs); a compute span followed by a TP
// collective runs as one iteration (plan flag 0x10). fin stores are 256-byte coalesced rows (32
// scenarios of one node), evict-first.
//
// Scheduling: every warp of the launch is co-resident (cudaLaunchCooperativeKernel refuses
// otherwise and the caller falls back to the level-by-level path), so a waiting warp cannot starve
// the producer it waits for. The build already proved the sync structure acyclic (plan.cpp) and the
// lockstep walk is deadlock-free because a cell's ranks are symmetric; a
// %globaltimer watchdog still turns any unexpected stall into PRISM_E_DEADLOCK instead of a hung
// GPU.
#include "cell_kernel.cuh"

#include <numeric>

namespace prism {

#ifdef PRISM_CELL_STATS
template <bool SH, bool PR, bool MS>
static const void *cell_kernel_tp(int tp, int ks) {
  if (ks == 16) {
    switch (tp) {
      case 2: return (const void *)cell_kernel<2, SH, PR, MS, 16>;
      case 4: return (const void *)cell_kernel<4, SH, PR, MS, 16>;
      default: return nullptr;
    }
  }
  if (ks == 8) {
    switch (tp) {
      case 2: return (const void *)cell_kernel<2, SH, PR, MS, 8>;
      case 4: return (const void *)cell_kernel<4, SH, PR, MS, 8>;
      case 8: return (const void *)cell_kernel<8, SH, PR, MS, 8>;
      default: return nullptr;
    }
  }
  switch (tp) {
    case 1: return (const void *)cell_kernel<1, SH, PR, MS>;
    case 2: return (const void *)cell_kernel<2, SH, PR, MS>;
    case 3: return (const void *)cell_kernel<3, SH, PR, MS>;
    case 4: return (const void *)cell_kernel<4, SH, PR, MS>;
    case 5: return (const void *)cell_kernel<5, SH, PR, MS>;
    case 6: return (const void *)cell_kernel<6, SH, PR, MS>;
    case 7: return (const void *)cell_kernel<7, SH, PR, MS>;
    case 8: return (const void *)cell_kernel<8, SH, PR, MS>;
    default: return nullptr;
  }
}
const void *cell_kernel_get(int tp, bool sh, bool pr, bool ms, int ks) {
  const int v = (sh ? 1 : 0) | (pr ? 2 : 0) | (ms ? 4 : 0);
  switch (v) {
    case 0: return cell_kernel_tp<false, false, false>(tp, ks);
    case 1: return cell_kernel_tp<true, false, false>(tp, ks);
    case 2: return cell_kernel_tp<false, true, false>(tp, ks);
    case 3: return cell_kernel_tp<true, true, false>(tp, ks);
    case 4: return cell_kernel_tp<false, false, true>(tp, ks);
    case 5: return cell_kernel_tp<true, false, true>(tp, ks);
    case 6: return cell_kernel_tp<false, true, true>(tp, ks);
    default: return cell_kernel_tp<true, true, true>(tp, ks);
  }
}
#endif

namespace {


// Kernel pointer of the graph's variant (type-erased: the variants are instantiated in the
// cells_k_*.cu units, compiled in parallel; PRISM_CELL_STATS builds instantiate them here so the
// statistics arrays are one set).
const void *cell_kernel_for(const DevGraph &g) {
  // cell width: the tp ranks of a TP cell, or the R replicas of a replica cell
  return cell_kernel_get(g.cell_R > 1 ? g.cell_R : g.tp, g.n_shards > 1, g.per_rank_dur != 0, g.ms != 0,
                         g.cta_ks > 1 ? g.cta_ks : 1);
}
// dynamic shared memory of the multi-stream state (0 otherwise)
size_t cell_dyn_smem(const DevGraph &g) {
  const int w = g.cell_R > 1 ? g.cell_R : g.tp, ks = g.cta_ks > 1 ? g.cta_ks : 1;
  const size_t msb = g.ms ? (size_t)(g.ms_streams + g.ms_events) * w * 32 * 8 * ks : 0;
  if (ks == 1) return msb;
  size_t per = 0;
  switch (w) {  // EP CTAs: per-warp scratch + the partial-max buffer, in dynamic shared memory
    case 2: per = cta_warp_scratch<2>(); break;
    case 4: per = cta_warp_scratch<4>(); break;
    default: per = cta_warp_scratch<8>(); break;
  }
  return (size_t)ks * per + 2 * (size_t)ks * 32 * 8 + msb;
}

cudaError_t preload_cell_kernels() {
  cudaFuncAttributes a;
  for (int tp = 1; tp <= MAX_TP; ++tp)
    for (int ks : {1, 8, 16})
      for (int v = 0; v < 8; ++v) {
        const void *f = cell_kernel_get(tp, v & 1, v & 2, v & 4, ks);
        if (!f) continue;
        cudaError_t e = cudaFuncGetAttributes(&a, f);
        if (e != cudaSuccess) return e;
        // allow the multi-stream state / the EP CTAs' scratch beyond the 48 KB default
        e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, ks > 1 ? 200 * 1024 : 96 * 1024);
        if (e != cudaSuccess) return e;
      }
  return cudaSuccess;
}

// CTAs needed for `units` warps, if they can all be co-resident.
bool cell_fit_units(const DevGraph &g, int64_t units, int *ctas) {
  const void *fn = cell_kernel_for(g);
  if (!fn) return false;  // tp > 8: the level-by-level schedule
  int dev = 0, sms = 0, coop = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return false;
  const int ks = g.cta_ks > 1 ? g.cta_ks : 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, ks * 32, cell_dyn_smem(g)) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const int64_t need = units;  // one CTA per unit (a cell, or the KS cells of an EP CTA)
  if (ctas) *ctas = (int)need;
  return need >= 1 && (int64_t)per_sm * sms >= need;
}

}  // namespace

cudaError_t preload_cells() { return preload_cell_kernels(); }

// Poll/backoff policy of the waiting warps; PRISM_POLL="spin,sleep0,sleep_max" overrides it
// (tuning experiments, tools/poll_sweep.py).
// PRISM_POLL_FAST="spin,sleep0,sleep_max" the fast wait's (sleep_max 0 turns it off).
struct PollPolicy {
  uint32_t spin, sleep0, sleep_max;
  uint32_t fspin, fsleep0, fsleep_max;
  uint32_t lean;
};
PollPolicy poll_policy() {
  PollPolicy p{2, 32, 1024, 4, 32, 256, 1};
  if (const char *e = std::getenv("PRISM_LEAN")) p.lean = (uint32_t)std::atoi(e);
  if (const char *e = std::getenv("PRISM_POLL")) {
    unsigned a = 0, b = 0, c = 0;
    if (std::sscanf(e, "%u,%u,%u", &a, &b, &c) == 3) p.spin = a, p.sleep0 = b, p.sleep_max = c;
  }
  if (const char *e = std::getenv("PRISM_POLL_FAST")) {
    unsigned a = 0, b = 0, c = 0;
    if (std::sscanf(e, "%u,%u,%u", &a, &b, &c) == 3) p.fspin = a, p.fsleep0 = b, p.fsleep_max = c;
  }
  return p;
}

// Chunks of 32 scenarios per unit; every chunk of a replay runs in one launch when they all fit,
// else the caller launches one chunk at a time (chunk groups of 1).
// CTAs of one chunk: cells, or EP CTAs of cta_ks cells
int64_t cell_count(const DevGraph &g) {
  return (int64_t)(g.s1 - g.s0) * (g.d1 - g.d0) / (g.cell_R > 1 ? g.cell_R : 1) / (g.cta_ks > 1 ? g.cta_ks : 1);
}

bool cells_fit(const DevGraph &g, int nchunks, int group) {
  return cell_fit_units(g, cell_count(g) * group, nullptr) && nchunks >= 1;
}

int cells_chunk_scenarios() { return SC; }

int cells_chunks_per_launch(const DevGraph &g, int nchunks, int group) {
  for (int c = nchunks; c > 1; --c)
    if (nchunks % c == 0 && cell_fit_units(g, cell_count(g) * c * group, nullptr)) return c;
  return 1;
}

cudaError_t launch_cells(const DevGraph &g, const ScenParams &p, int64_t *rslot, int64_t *acc,
                         int64_t *rres, uint32_t *arrive, uint32_t *status, int parity, int64_t *fin,
                         int64_t *gfin, int64_t *rank_end, int chunk0, int nchunks_launch, int Sp,
                         const ShardLink *link, cudaStream_t st) {
  // a local-group launch (link->lg shards of this device) covers every shard's cells
  const int64_t units = cell_count(g) * nchunks_launch * (link && link->lg > 0 ? link->lg : 1);
  int ctas = 0;
  if (!cell_fit_units(g, units, &ctas)) return cudaErrorCooperativeLaunchTooLarge;
  // the launch covers chunks [chunk0, chunk0 + nchunks_launch) of the replay's Sp / 32 chunks
  static const PollPolicy pol = poll_policy();
  CellArgs a{rslot, acc, rres, arrive, status, g.watchdog_ns, parity, (int32_t)units, Sp, chunk0,
             Sp / SC, pol.spin, pol.sleep0, pol.sleep_max, pol.fspin, pol.fsleep0, pol.fsleep_max, pol.lean, 1u, ShardLink{}};
  {  // CTA -> cell placement: CTAs are dealt to the SMs in index order, and with the identity map
     // an SM holds warps of only a few pipeline stages (whose busy and idle phases coincide in a
     // 1F1B schedule); a permutation of the cells by a stride coprime with their count mixes the
     // stages per SM (C5 cell kernel 2.66 -> 2.58 ms, any of 16 strides tried within noise of each
     // other, tools/exp/mix_sweep.sh). PRISM_CELL_MIX overrides it (1 = identity).
    static const uint32_t mix = [] {
      const char *e = std::getenv("PRISM_CELL_MIX");
      return e ? (uint32_t)std::atoi(e) : 257u;
    }();
    const int64_t cells = units / nchunks_launch / (link && link->lg > 0 ? link->lg : 1);
    if (mix > 1 && std::gcd((int64_t)mix, cells) == 1) a.mix = mix;
  }
  if (link) a.L = *link;
  DevGraph gg = g;
  ScenParams pp = p;
  int64_t *fin_g = fin;
  void *args[] = {&gg, &pp, &a, &fin_g, &gfin, &rank_end};
  return cudaLaunchCooperativeKernel(cell_kernel_for(g), dim3(ctas), dim3((g.cta_ks > 1 ? g.cta_ks : 1) * 32), args,
                                     cell_dyn_smem(g), st);
}

// Debug statistics of the last cell-kernel launch (PRISM_CELL_STATS builds only).
extern "C" PRISM_API int prism_debug_lat(unsigned long long *out) {
#ifdef PRISM_CELL_STATS
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_lat, sizeof(unsigned long long) * 4);
  unsigned long long z[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(g_lat, z, sizeof z);
  return 0;
#else
  (void)out;
  return -2;
#endif
}

extern "C" PRISM_API int prism_debug_timeline(unsigned long long *out) {
#ifdef PRISM_CELL_STATS
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, g_tl, sizeof(unsigned long long) * 16 * 128 * 4) == cudaSuccess ? 0 : -1;
#else
  (void)out;
  return -2;
#endif
}

extern "C" PRISM_API int prism_debug_wait_hist(unsigned long long *out) {
#ifdef PRISM_CELL_STATS
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, g_wait_hist, sizeof(unsigned long long) * 16 * 4096) != cudaSuccess) return -1;
  static unsigned long long zeros[16 * 4096];
  cudaMemcpyToSymbol(g_wait_hist, zeros, sizeof zeros);
  return 0;
#else
  (void)out;
  return -2;
#endif
}

extern "C" PRISM_API int prism_debug_cell_stats(unsigned long long *out, int n) {
#ifdef PRISM_CELL_STATS
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, g_cell_stats, sizeof(unsigned long long) * (size_t)n) != cudaSuccess) return -1;
  static unsigned long long zeros[16384 * 8];
  cudaMemcpyToSymbol(g_cell_stats, zeros, sizeof zeros);
  return 0;
#else
  (void)out;
  (void)n;
  return -2;
#endif
}

}  // namespace prism
