// replay_cells.cu — replay v2: one persistent cooperative launch for the whole replay (rows a6-a8).
//
// Same semantics as replay.cu (readings Z2-Z5), different
// schedule. A *cell* is one TP group: the tp ranks of a (stage, dp) pair. They run the same stage
// template, so they walk it in lockstep, and every TP collective's members are exactly
// the cell. One CTA owns one (cell, 64-scenario chunk): ceil(tp/2) warps, each warp = two of
// the cell's ranks (half-warps), each lane = 4 scenarios of its rank (warp-cooperative per-rank op
// chains, 4 independent hash chains per lane). Per op:
//   compute span      : t += dur'                               (registers only)
//   TP collective     : segmented max over the cell's ranks through shared memory (one
//                       __syncthreads, double-buffered slots), t = max + dur'_g
//   small cross-cell  : (P2P message, EP/EDP group of <= 8) every member stores its ready times
//   group               into its global ready slot (reset to -1 before the launch) and polls the
//                       other members' slots until they are valid: an aligned 8-byte store is
//                       single-copy atomic, so the value is its own flag and no fence is needed
//   large cross-cell  : (DP, WORLD, big EP) red.max of the ready times into the group's
//   group               accumulator, fence, arrive on its counter; members poll the counter and
//                       read the accumulator (segmented max done by the L2 atomics)
// and a node finishes at the max over its groups' (start + dur'_g) (reading Z3).
// Scheduling: every CTA of a 64-scenario chunk is co-resident (cudaLaunchCooperativeKernel refuses
// otherwise and the caller falls back to the level-by-level path), so a waiting warp cannot starve
// the producer it waits for; chunks run as successive launches. The build already proved the sync
// structure acyclic (plan.cpp) and the lockstep walk is deadlock-free because a cell's ranks are
// symmetric; a %globaltimer watchdog still turns any unexpected stall into
// PRISM_E_DEADLOCK instead of a hung GPU.
#include <cuda_runtime.h>

#include <algorithm>

#include "graph.h"

namespace prism {

namespace {

#ifndef PRISM_CELL_MINB
#define PRISM_CELL_MINB 7
#endif
constexpr uint64_t K_GOLD = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t K_MIX = 0xBF58476D1CE4E5B9ULL;
constexpr int SPL = 4;        // scenarios per lane
constexpr int SC = 16 * SPL;  // scenarios per unit (a half-warp covers one rank)
constexpr int MAX_TP = 8;     // CTA = ceil(tp/2) warps <= 128 threads
constexpr int SMALL = kSmallGroup;  // groups up to this size use the value-as-flag protocol

__device__ __forceinline__ int64_t perturb_x(int64_t d, uint64_t x, const ScenParams &p) {
  const uint64_t h = splitmix64(x);
  const uint32_t v = (uint32_t)(h >> 40);
  const uint64_t low = p.mod_magic * (uint64_t)v;
  const uint32_t r = (uint32_t)__umul64hi(low, (uint64_t)(uint32_t)p.mod);
  const int64_t delta = (int64_t)r - p.amp;
  return (d * (65536 + delta)) >> 16;
}

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
__device__ __forceinline__ void ld_relaxed4(const int64_t *p, int64_t *v) {
  asm volatile("ld.relaxed.gpu.global.v2.s64 {%0, %1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "l"(p) : "memory");
  asm volatile("ld.relaxed.gpu.global.v2.s64 {%0, %1}, [%2];" : "=l"(v[2]), "=l"(v[3]) : "l"(p + 2) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st4(int64_t *p, const int64_t *t) {
  *reinterpret_cast<longlong2 *>(p) = make_longlong2(t[0], t[1]);
  *reinterpret_cast<longlong2 *>(p + 2) = make_longlong2(t[2], t[3]);
}
__device__ __forceinline__ void red_max(int64_t *p, int64_t v) {
  asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"((uint64_t)v) : "memory");
}

struct CellArgs {
  int64_t *rslot;      // [M_cross][Sp] ready slots of small-group memberships
  int64_t *acc;        // [G_large][Sp] max-accumulators of large groups (zeroed per replay)
  uint32_t *arrive;    // [G_large] arrival counters of large groups (zeroed per replay)
  uint32_t *status;    // [0] = abort flag / error code
  uint64_t timeout_ns;
  int32_t parity;      // ready-slot encoding of this replay: 0 -> t (valid >= 0), 1 -> ~t (valid < 0);
                       // every slot is written once per replay, so the previous replay's values
                       // read as "not yet" and no reset pass is needed
};

__device__ __forceinline__ int32_t rank_of(const DevGraph &g, int32_t tp_i, int32_t pp_i, int32_t dp_i) {
  return g.order == PRISM_ORDER_MEGATRON ? tp_i + g.tp * (dp_i + g.dp * pp_i)
                                         : tp_i + g.tp * (pp_i + g.pp * dp_i);
}

// Backoff + watchdog for a waiting lane; returns true when the replay was aborted.
__device__ __forceinline__ bool wait_tick(const CellArgs &a, uint32_t &spins, uint64_t &t0) {
  ++spins;
  __nanosleep(spins < 8 ? 20u * spins : 200u);
  if ((spins & 255) == 0) {
    if (ld_relaxed(a.status) != 0) return true;
    if (t0 == 0) t0 = globaltimer();
    if (globaltimer() - t0 > a.timeout_ns) {
      atomicCAS(a.status, 0u, (uint32_t)PRISM_E_DEADLOCK);
      return true;
    }
  }
  return false;
}

// Cross-cell synchronization of node n for this lane's 4 scenarios (t = ready on entry, finish on
// exit). Returns false when the watchdog aborted the replay.
__device__ __forceinline__ bool cross_sync(const DevGraph &g, const ScenParams &p, const CellArgs &a,
                                           int64_t *__restrict__ gfin, int32_t n, int32_t k0, int32_t Sp,
                                           bool active, bool lead, int64_t *t) {
  const int32_t h0 = g.node_gptr[n], h1 = g.node_gptr[n + 1];
  // 1. arrive on every group of the node
  bool large_any = false;
  for (int32_t h = h0; h < h1; ++h) {
    const int32_t gg = g.node_grp[h];
    const int32_t mb = g.grp_ptr[gg], size = g.grp_ptr[gg + 1] - mb;
    if (size <= SMALL) {
      if (active) {
        int64_t v[SPL];
#pragma unroll
        for (int q = 0; q < SPL; ++q) v[q] = a.parity ? ~t[q] : t[q];
        st4(a.rslot + (g.grp_xbase[gg] + (g.node_mslot[h] - mb)) * Sp + k0, v);
      }
    } else {
      large_any = true;
      if (active)
        for (int q = 0; q < SPL; ++q) red_max(a.acc + (int64_t)g.grp_lidx[gg] * Sp + k0 + q, t[q]);
    }
  }
  if (large_any) {
    __threadfence();  // the accumulations are performed before the arrival is counted
    __syncwarp();
    if (lead)
      for (int32_t h = h0; h < h1; ++h) {
        const int32_t gg = g.node_grp[h];
        if (g.grp_ptr[gg + 1] - g.grp_ptr[gg] > SMALL) atomicAdd(a.arrive + g.grp_lidx[gg], 1u);
      }
  }
  // 2. wait for every group, finish = max over groups of (max ready + dur')
  int64_t f[SPL] = {0, 0, 0, 0};
  const uint64_t sx = p.seed;
  uint32_t spins = 0;
  uint64_t tw = 0;
  for (int32_t h = h0; h < h1; ++h) {
    const int32_t gg = g.node_grp[h];
    const int32_t mb = g.grp_ptr[gg], size = g.grp_ptr[gg + 1] - mb;
    int64_t m[SPL] = {0, 0, 0, 0};
    if (size <= SMALL) {
      const int64_t xb = g.grp_xbase[gg];
      for (int32_t mm = 0; mm < size; ++mm) {
        int64_t v[SPL];
        const int64_t *src = a.rslot + (xb + mm) * Sp + k0;
        while (true) {
          ld_relaxed4(src, v);
          const int64_t all = a.parity ? (v[0] & v[1] & v[2] & v[3]) : (v[0] | v[1] | v[2] | v[3]);
          if ((a.parity ? all < 0 : all >= 0) || !active) break;
          if (wait_tick(a, spins, tw)) return false;
        }
        for (int q = 0; q < SPL; ++q) m[q] = max(m[q], a.parity ? ~v[q] : v[q]);
      }
    } else {
      // chunks run as successive launches and every chunk adds `size` arrivals
      const uint32_t *cnt = a.arrive + g.grp_lidx[gg];
      while (ld_relaxed(cnt) < (uint32_t)size * (uint32_t)(k0 / SC + 1)) {
        if (wait_tick(a, spins, tw)) return false;
      }
      fence_acq_rel();
      const int64_t *src = a.acc + (int64_t)g.grp_lidx[gg] * Sp + k0;
      for (int q = 0; q < SPL; ++q) m[q] = __ldcg(src + q);
    }
    const int64_t gd = g.grp_dur[gg];
    const uint64_t uid = g.grp_uid[gg];
    const uint32_t gb = (uid >> 56) == PRISM_ROLE_P2P ? 4u : 2u;
    const bool gp = (p.mask & gb) && p.amp > 0;
    const uint64_t gx = uid * K_MIX;
    int64_t e[SPL];
#pragma unroll
    for (int q = 0; q < SPL; ++q) {
      const int32_t k = k0 + q;
      e[q] = (gp && k > 0) ? perturb_x(gd, sx ^ ((uint64_t)k * K_GOLD) ^ gx, p) : gd;
      m[q] += e[q];
      f[q] = max(f[q], m[q]);
    }
    // the group's finish is kept for queries of multi-group (P2P batch) nodes; every member
    // computes the same value, so a node with several groups stores its own groups' finishes
    if (active && h1 - h0 > 1) st4(gfin + (int64_t)gg * Sp + k0, m);
  }
#pragma unroll
  for (int q = 0; q < SPL; ++q) t[q] = f[q];
  return true;
}

__global__ void __launch_bounds__(128, PRISM_CELL_MINB) cell_kernel(DevGraph g, ScenParams p, CellArgs a,
                                                                   int32_t chunk, int32_t Sp,
                                                                   int64_t *__restrict__ fin,
                                                                   int64_t *__restrict__ gfin,
                                                                   int64_t *__restrict__ rank_end) {
  __shared__ __align__(16) int64_t slot[2][MAX_TP][16][SPL];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, l16 = lane & 15;
  const int32_t tpi = 2 * w + half;
  const bool active = tpi < g.tp;
  const int32_t cell = blockIdx.x;
  const int32_t s = cell % g.pp, dpi = cell / g.pp;
  const int32_t r = rank_of(g, active ? tpi : 0, s, dpi);
  const int32_t rb = g.rank_ptr[r];
  const int32_t len = g.rank_ptr[r + 1] - rb;
  const int32_t k0 = chunk * SC + l16 * SPL;
  const bool lead = l16 == 0 && active;
  const bool cpert = (p.mask & 1u) && p.amp > 0;
  const bool gpert = (p.mask & 2u) && p.amp > 0;
  uint64_t sx[SPL];
  bool pj[SPL];
#pragma unroll
  for (int q = 0; q < SPL; ++q) {
    sx[q] = p.seed ^ ((uint64_t)(k0 + q) * K_GOLD);
    pj[q] = k0 + q > 0;
  }
  int64_t t[SPL] = {0, 0, 0, 0};
  int buf = 0;
  for (int32_t base = 0; base < len; base += 16) {
    // one coalesced round trip for the next 16 ops of each of the warp's two ranks
    const int32_t cnt = min(16, len - base);
    uint32_t cls = 2;
    int64_t dl = 0;
    uint64_t uxl = 0;
    if (l16 < cnt) {
      const int32_t n = rb + base + l16;
      cls = g.node_cls[n];
      dl = g.node_sdur[n];
      uxl = g.node_uid[n] * K_MIX;
    }
    for (int32_t j = 0; j < cnt; ++j) {
      const int src = (half << 4) | j;
      const uint32_t c = __shfl_sync(0xffffffffu, cls, src);
      const int64_t d = __shfl_sync(0xffffffffu, dl, src);
      const uint64_t ux = __shfl_sync(0xffffffffu, uxl, src);
      const int32_t n = rb + base + j;
      if (c == 0) {  // compute span: wait out the (perturbed) duration
        if (cpert) {
#pragma unroll
          for (int q = 0; q < SPL; ++q) t[q] += pj[q] ? perturb_x(d, sx[q] ^ ux, p) : d;
        } else {
#pragma unroll
          for (int q = 0; q < SPL; ++q) t[q] += d;
        }
      } else if (c == 1) {  // in-cell TP collective: segmented max over the cell's ranks
        int64_t e[SPL];
#pragma unroll
        for (int q = 0; q < SPL; ++q) e[q] = (gpert && pj[q]) ? perturb_x(d, sx[q] ^ ux, p) : d;
        if (active) {
          *reinterpret_cast<longlong2 *>(&slot[buf][tpi][l16][0]) = make_longlong2(t[0], t[1]);
          *reinterpret_cast<longlong2 *>(&slot[buf][tpi][l16][2]) = make_longlong2(t[2], t[3]);
        }
        __syncthreads();
        int64_t m[SPL] = {0, 0, 0, 0};
        for (int qq = 0; qq < g.tp; ++qq) {
          const longlong2 v0 = *reinterpret_cast<const longlong2 *>(&slot[buf][qq][l16][0]);
          const longlong2 v1 = *reinterpret_cast<const longlong2 *>(&slot[buf][qq][l16][2]);
          m[0] = max(m[0], (int64_t)v0.x);
          m[1] = max(m[1], (int64_t)v0.y);
          m[2] = max(m[2], (int64_t)v1.x);
          m[3] = max(m[3], (int64_t)v1.y);
        }
        buf ^= 1;
#pragma unroll
        for (int q = 0; q < SPL; ++q) t[q] = m[q] + e[q];
      } else {  // cross-cell synchronization
        if (!cross_sync(g, p, a, gfin, n, k0, Sp, active, lead, t)) return;
      }
      if (p.record && active) st4(fin + (int64_t)n * Sp + k0, t);
    }
  }
  if (active) st4(rank_end + (int64_t)r * Sp + k0, t);
}

bool cell_fit(const DevGraph &g) {
  if (g.tp > MAX_TP) return false;
  const int threads = ((g.tp + 1) / 2) * 32;
  int dev = 0, sms = 0, coop = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return false;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cell_kernel, threads, 0) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return (int64_t)per_sm * sms >= (int64_t)g.pp * g.dp;
}

}  // namespace

bool cells_fit(const DevGraph &g, int nchunks) {
  (void)nchunks;  // chunks run as successive launches
  return cell_fit(g);
}

int cells_chunk_scenarios() { return SC; }

cudaError_t launch_cells(const DevGraph &g, const ScenParams &p, int64_t *rslot, int64_t *acc,
                         uint32_t *arrive, uint32_t *status, int parity, int64_t *fin, int64_t *gfin,
                         int64_t *rank_end, int chunk, int Sp, cudaStream_t st) {
  if (!cell_fit(g)) return cudaErrorCooperativeLaunchTooLarge;
  CellArgs a{rslot, acc, arrive, status, 10ull * 1000 * 1000 * 1000, parity};
  DevGraph gg = g;
  ScenParams pp = p;
  int32_t ch = chunk, sp = Sp;
  void *args[] = {&gg, &pp, &a, &ch, &sp, &fin, &gfin, &rank_end};
  return cudaLaunchCooperativeKernel((const void *)cell_kernel, dim3(g.pp * g.dp), dim3(((g.tp + 1) / 2) * 32),
                                     args, 0, st);
}

}  // namespace prism
