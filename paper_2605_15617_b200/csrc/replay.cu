// replay.cu — rows a6-a8: wavefront replay over the level-sorted CSR DAG.
//
// Semantics (§5.1, §6.1, §5.3; readings Z2-Z5 in DESIGN.md §3):
//   ready(n)  = finish of n's stream predecessor (0 for a rank's first op)
//   compute   : finish = ready + dur'                              (waits out the duration)
//   group g   : start_g = max over members of ready (segmented max); gfin_g = start_g + dur'_g
//   sync node : finish = max over its groups of gfin_g              (all must reach it)
// One launch per frontier level l (row a5) relaxes every group of level l: for each membership a
// team of L lanes (lane = scenario, SPL scenarios per lane) walks the member's chain segment from
// its previous sync node (resolved at a lower level) through the compute spans in between,
// writing their finish times (once, by the membership in the node's first slot), and folds the
// member's ready time into a shared-memory accumulator of its group (the segmented max); the
// block then writes gfin for its groups. All arithmetic is int64; results are exact.
#include <cuda_runtime.h>

#include <algorithm>

#include "graph.h"

namespace prism {

namespace {

constexpr uint64_t K_GOLD = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t K_MIX = 0xBF58476D1CE4E5B9ULL;

// Reading Z8: d' = (d * (65536 + delta)) >> 16, delta = ((h >> 40) mod (2 amp + 1)) - amp with
// h = splitmix64(seed ^ k*K_GOLD ^ uid*K_MIX). `x` is that xor already formed. The mod uses
// Lemire's direct remainder (exact for 32-bit numerators): r = hi64((M * v) mod 2^64, d).

template <int SPL>
struct Vec;
template <>
struct Vec<1> {
  __device__ static void store(int64_t *p, const int64_t *t) { *p = t[0]; }
  __device__ static void load_max(const int64_t *p, int64_t *t) { t[0] = max(t[0], __ldcg(p)); }
};
template <>
struct Vec<2> {
  __device__ static void store(int64_t *p, const int64_t *t) {
    longlong2 v;
    v.x = t[0];
    v.y = t[1];
    *reinterpret_cast<longlong2 *>(p) = v;
  }
  __device__ static void load_max(const int64_t *p, int64_t *t) {
    longlong2 v = __ldcg(reinterpret_cast<const longlong2 *>(p));
    t[0] = max(t[0], (int64_t)v.x);
    t[1] = max(t[1], (int64_t)v.y);
  }
};

// Walk the chain segment that ends at node n: returns ready(n) per scenario in t[]. When `write`,
// stores the finish of the previous sync node and of every compute span in the segment.
template <int SPL>
__device__ __forceinline__ void walk_segment(const DevGraph &g, const ScenParams &p, int32_t r,
                                             int32_t ps, int32_t end, int64_t *__restrict__ fin,
                                             const int64_t *__restrict__ gfin, int32_t Sp, int32_t k0,
                                             const uint64_t *sx, const bool *pj, bool write, int64_t *t) {
  const int32_t rb = g.rank_ptr[r];
#pragma unroll
  for (int j = 0; j < SPL; ++j) t[j] = 0;
  if (ps >= 0) {
    const int32_t h0 = g.node_gptr[ps], h1 = g.node_gptr[ps + 1];
    for (int32_t h = h0; h < h1; ++h) {
      const int64_t grp = g.node_grp[h];
      Vec<SPL>::load_max(gfin + grp * Sp + k0, t);
    }
    if (write) Vec<SPL>::store(fin + fin_off(g, fin_row(g, ps), k0, Sp), t);
  }
  const uint64_t rhi = (uint64_t)r << 32;
  for (int32_t i = (ps >= 0 ? ps + 1 : rb); i < end; ++i) {
    const int64_t d = nd_dur(g, i);
    const uint64_t uidx = (rhi | (uint32_t)(i - rb)) * K_MIX;
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      const int64_t dd = pj[j] ? perturb_x(d, sx[j] ^ uidx, p) : d;
      t[j] += dd;
    }
    if (write) Vec<SPL>::store(fin + fin_off(g, fin_row(g, i), k0, Sp), t);
  }
}

template <int L, int SPL>
__global__ void __launch_bounds__(256) level_kernel(DevGraph g, ScenParams p,
                                                     const Tile *__restrict__ tiles,
                                                     int64_t *__restrict__ fin,
                                                     int64_t *__restrict__ gfin) {
  constexpr int SC = L * SPL;
  constexpr int TEAMS = 256 / L;
  extern __shared__ unsigned long long acc[];
  const Tile tl = tiles[blockIdx.x];
  const QGroup &q = g.q[tl.q];
  const int32_t z = q.size;
  const int32_t cnt = tl.cnt;
  const int64_t g0 = q.gbase + tl.i0;
  const int64_t m0 = q.mbase + (int64_t)tl.i0 * z;
  const int32_t nmem = cnt * z;
  const int32_t Sp = gridDim.y * SC;
  // the frontier tile's member list (a contiguous run of grp_mem) is staged in shared memory by a
  // TMA bulk copy, completed on an mbarrier, while the threads clear the accumulators; a tile of a
  // huge group (> kTileMem members) reads its members from global memory instead
  constexpr int kTileMem = 512;
  __shared__ __align__(16) int32_t mem_s[kTileMem + 8];
  __shared__ __align__(8) uint64_t bar;
  const int64_t a0 = m0 & ~(int64_t)3, a1 = (m0 + nmem + 3) & ~(int64_t)3;  // 16-byte aligned superset
  const bool staged = a1 - a0 <= kTileMem + 8;
  if (staged && threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (uint32_t)((a1 - a0) * 4));
    tma_load_1d(mem_s, g.grp_mem + a0, (uint32_t)((a1 - a0) * 4), &bar);
  }
  for (int x = threadIdx.x; x < cnt * SC; x += 256) acc[x] = 0ULL;
  __syncthreads();
  if (staged) mbar_wait(&bar, 0);
  const int32_t *mem = staged ? mem_s + (m0 - a0) : g.grp_mem + m0;

  const int team = threadIdx.x / L, lane = threadIdx.x % L;
  const int32_t k0 = blockIdx.y * SC + lane * SPL;
  uint64_t sx[SPL];
  bool pj[SPL];  // scenario 0 and unmasked kinds are never perturbed
#pragma unroll
  for (int j = 0; j < SPL; ++j) {
    sx[j] = p.seed ^ ((uint64_t)(p.first + k0 + j) * K_GOLD);
    pj[j] = (p.mask & 1u) && p.amp > 0 && (p.first + k0 + j) > 0;
  }
  for (int32_t mm = team; mm < nmem; mm += TEAMS) {
    const int32_t n = mem[mm];
    const int32_t gl = mm / z;
    const int32_t r = g.node_rank[n];
    const int32_t ps = g.node_prev_sync[n];
    const bool primary = p.record && g.node_grp[g.node_gptr[n]] == (int32_t)(g0 + gl);
    int64_t t[SPL];
    walk_segment<SPL>(g, p, r, ps, n, fin, gfin, Sp, k0, sx, pj, primary, t);
#pragma unroll
    for (int j = 0; j < SPL; ++j) atomicMax(&acc[gl * SC + lane * SPL + j], (unsigned long long)t[j]);
  }
  __syncthreads();
  const uint32_t gbit = q.type == PRISM_ROLE_P2P ? 4u : 2u;
  const bool gpert = (p.mask & gbit) && p.amp > 0;
  for (int x = threadIdx.x; x < cnt * SC; x += 256) {
    const int32_t gl = x / SC;
    const int32_t kk = blockIdx.y * SC + (x - gl * SC);
    const int64_t grp = g0 + gl;
    const int64_t d = g.grp_dur[grp];
    int64_t dd = d;
    const int32_t kg = p.first + kk;  // global scenario index (perturbation key)
    if (gpert && kg > 0) dd = perturb_x(d, p.seed ^ ((uint64_t)kg * K_GOLD) ^ (g.grp_uid[grp] * K_MIX), p);
    gfin[grp * Sp + kk] = (int64_t)acc[x] + dd;
  }
}

// Tail: after the last sync node of every rank (or the whole chain if it has none).
template <int L, int SPL>
__global__ void __launch_bounds__(256) tail_kernel(DevGraph g, ScenParams p, int64_t *__restrict__ fin,
                                                    const int64_t *__restrict__ gfin,
                                                    int64_t *__restrict__ rank_end) {
  constexpr int SC = L * SPL;
  constexpr int TEAMS = 256 / L;
  const int32_t Sp = gridDim.y * SC;
  const int team = threadIdx.x / L, lane = threadIdx.x % L;
  const int32_t k0 = blockIdx.y * SC + lane * SPL;
  uint64_t sx[SPL];
  bool pj[SPL];
#pragma unroll
  for (int j = 0; j < SPL; ++j) {
    sx[j] = p.seed ^ ((uint64_t)(p.first + k0 + j) * K_GOLD);
    pj[j] = (p.mask & 1u) && p.amp > 0 && (p.first + k0 + j) > 0;
  }
  for (int32_t r = blockIdx.x * TEAMS + team; r < g.W; r += gridDim.x * TEAMS) {
    const int32_t rb = g.rank_ptr[r], re = g.rank_ptr[r + 1];
    int64_t t[SPL];
    if (re == rb) {
#pragma unroll
      for (int j = 0; j < SPL; ++j) t[j] = 0;
    } else {
      const int32_t last = re - 1;
      const bool last_sync = g.node_gptr[last + 1] > g.node_gptr[last];
      const int32_t ps = last_sync ? last : g.node_prev_sync[last];
      walk_segment<SPL>(g, p, r, ps, re, fin, gfin, Sp, k0, sx, pj, p.record != 0, t);
    }
    Vec<SPL>::store(rank_end + (int64_t)r * Sp + k0, t);
  }
}

// Row a8: T_k = max over ranks of the rank's last finish (every chain is non-decreasing).
// Row a8: iteration time of each scenario = max over ranks of rank_end[r][k] (all >= 0). Block
// (x, y): 32 consecutive scenarios (coalesced 256-byte rows) x 8 rank lanes, ranks strided over
// grid.y; a shared-memory max over the 8 rank lanes, then one atomicMax per scenario into iter,
// which the launcher zeroes first.
__global__ void __launch_bounds__(256) reduce_iter_kernel(int32_t W, int32_t S, int32_t Sp,
                                                          const int64_t *__restrict__ rank_end,
                                                          int64_t *__restrict__ iter) {
  const int kx = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int32_t k = blockIdx.x * 32 + kx;
  int64_t m = 0;
  if (k < Sp)
    for (int32_t r = blockIdx.y * 8 + ry; r < W; r += gridDim.y * 8) m = max(m, rank_end[(int64_t)r * Sp + k]);
  __shared__ int64_t sm[8][32];
  sm[ry][kx] = m;
  __syncthreads();
  if (ry == 0) {
#pragma unroll
    for (int y = 1; y < 8; ++y) m = max(m, sm[y][kx]);
    if (k < S) atomicMax((unsigned long long *)(iter + k), (unsigned long long)m);
  }
}

// Row e, sharded replay: partial iteration time of this shard's ranks (one block per scenario).
__global__ void __launch_bounds__(256) shard_partial_kernel(DevGraph g, int32_t Sp,
                                                            const int64_t *__restrict__ rank_end,
                                                            int64_t *__restrict__ part) {
  const int32_t k = blockIdx.x;
  const int32_t ns = g.s1 - g.s0;
  const int32_t nloc = g.tp * ns * (g.d1 - g.d0);
  int64_t m = 0;
  for (int32_t x = threadIdx.x; x < nloc; x += blockDim.x) {
    const int32_t tpi = x % g.tp, s = g.s0 + (x / g.tp) % ns, dpi = g.d0 + x / (g.tp * ns);
    const int32_t r = g.order == PRISM_ORDER_MEGATRON ? tpi + g.tp * (dpi + g.dp * s)
                                                      : tpi + g.tp * (s + g.pp * dpi);
    m = max(m, rank_end[(int64_t)r * Sp + k]);
  }
  for (int off = 16; off; off >>= 1) m = max(m, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)m, off));
  __shared__ int64_t wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = max(m, wm[w]);
    part[k] = max(m, wm[0]);
  }
}

// Row e, local-group launch (prism_replay_local_shards): every shard of the device wrote its own
// ranks' rank_end rows into its own array; T_k = max over shards and their ranks (one block per
// scenario).
__global__ void __launch_bounds__(256) local_group_reduce_kernel(DevGraph g, ShardLink L, int32_t Sp,
                                                                 int64_t *__restrict__ iter) {
  const int32_t k = blockIdx.x;
  const bool ppx = g.shard_axis == 1;
  const int32_t ns = ppx ? g.pp / g.n_shards : g.pp, nd = ppx ? g.dp : g.dp / g.n_shards;
  const int32_t nloc = g.tp * ns * nd;
  int64_t m = 0;
  for (int32_t sh = 0; sh < L.lg; ++sh) {
    const int64_t *re = L.lg_rank_end[sh];
    const int32_t s0 = ppx ? sh * ns : 0, d0 = ppx ? 0 : sh * nd;
    for (int32_t x = threadIdx.x; x < nloc; x += blockDim.x) {
      const int32_t tpi = x % g.tp, s = s0 + (x / g.tp) % ns, dpi = d0 + x / (g.tp * ns);
      const int32_t r = g.order == PRISM_ORDER_MEGATRON ? tpi + g.tp * (dpi + g.dp * s)
                                                        : tpi + g.tp * (s + g.pp * dpi);
      m = max(m, re[(int64_t)r * Sp + k]);
    }
  }
  for (int off = 16; off; off >>= 1) m = max(m, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)m, off));
  __shared__ int64_t wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = max(m, wm[w]);
    iter[k] = max(m, wm[0]);
  }
}

// Row e: exchange of the partials over peer memory, then T_k = max over shards. One block: store
// this shard's S partials into slot [epoch & 1][self] of every shard's buffer, fence (system
// scope), publish flag[self] = epoch at every shard, wait for every shard's flag, reduce. The two
// part buffers alternate by epoch: a shard can only reach replay e+2's exchange after every shard
// finished reading replay e's.
__global__ void __launch_bounds__(1024) shard_exchange_kernel(ShardLink L, int32_t S, int32_t Sp,
                                                              const int64_t *__restrict__ part,
                                                              int64_t *__restrict__ iter,
                                                              uint32_t *status, uint64_t watchdog_ns) {
  const int64_t slab = (int64_t)L.n * Sp;  // int64 per epoch-parity buffer
  const int64_t po = (int64_t)(L.epoch & 1) * slab + (int64_t)L.self * Sp;
  for (int m = 0; m < L.n; ++m) {
    int64_t *dst = (int64_t *)(L.base[m] + L.o_part) + po;
    for (int32_t k = threadIdx.x; k < S; k += blockDim.x) dst[k] = part[k];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < L.n) {
    uint32_t *f = (uint32_t *)(L.base[threadIdx.x] + L.o_flag) + L.self;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(L.epoch) : "memory");
  }
  __shared__ int aborted;
  if (threadIdx.x == 0) aborted = 0;
  __syncthreads();
  if (threadIdx.x < L.n) {
    const uint32_t *f = (const uint32_t *)(L.base[L.self] + L.o_flag) + threadIdx.x;
    uint64_t t0 = 0;
    uint32_t spins = 0;
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if ((int32_t)(v - L.epoch) >= 0) break;
      __nanosleep(200);
      if ((++spins & 255) == 0) {
        uint64_t now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        if (now - t0 > watchdog_ns) {
          atomicCAS(status, 0u, (uint32_t)PRISM_E_DEADLOCK);
          aborted = 1;
          break;
        }
      }
    }
  }
  __syncthreads();
  if (aborted) return;
  const int64_t *mine = (const int64_t *)(L.base[L.self] + L.o_part) + (int64_t)(L.epoch & 1) * slab;
  for (int32_t k = threadIdx.x; k < S; k += blockDim.x) {
    int64_t m = 0;
    for (int s = 0; s < L.n; ++s) m = max(m, __ldcv(mine + (int64_t)s * Sp + k));
    iter[k] = m;
  }
}

// Row e, prism_shard_gather: every shard writes its own ranks' finish times of scenario k (and the
// finishes of the batched-P2P groups whose first member it owns) into the gather columns of every
// shard's exchange buffer (rows in fin_row order, one scenario: Sp = 1 layout), over NVLink peer
// stores; a local-group launch (L.lg > 0) does it for every shard of the device at once.
__device__ __forceinline__ bool owns_rank(const DevGraph &g, int32_t r, int32_t sh) {
  const int32_t s = g.order == PRISM_ORDER_MEGATRON ? r / (g.tp * g.dp) : (r / g.tp) % g.pp;
  const int32_t dpi = g.order == PRISM_ORDER_MEGATRON ? (r / g.tp) % g.dp : r / (g.tp * g.pp);
  return g.shard_axis == 1 ? s / (g.pp / g.n_shards) == sh : dpi / (g.dp / g.n_shards) == sh;
}

__global__ void __launch_bounds__(256) gather_kernel(DevGraph g, ShardLink L, const int64_t *__restrict__ fin,
                                                     const int64_t *__restrict__ gfin, int32_t Sp, int32_t k) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int32_t nsrc = L.lg > 0 ? L.lg : 1;
  for (int32_t src = 0; src < nsrc; ++src) {
    const int32_t sh = L.lg > 0 ? src : L.self;
    const int64_t *f = L.lg > 0 ? L.lg_fin[src] : fin;
    const int64_t *gf = L.lg > 0 ? L.lg_gfin[src] : gfin;
    // the source shard's fin rows start at its own node0 (DP blocks under TP_PP_DP), else 0
    const int64_t node0 = (g.shard_axis == 0 && g.order == PRISM_ORDER_TP_PP_DP) ? (int64_t)sh * g.fin_rows : 0;
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < g.N; n += stride) {
      if (!owns_rank(g, g.node_rank[n], sh)) continue;
      const int64_t row = fin_row(g, (int32_t)n);
      const int64_t v = f[((int64_t)(k / (Sp < 32 ? Sp : 32)) * g.fin_rows + row - node0) * (Sp < 32 ? Sp : 32) +
                          k % (Sp < 32 ? Sp : 32)];
      for (int m = 0; m < L.n; ++m) ((int64_t *)(L.base[m] + L.o_gcol))[row] = v;
    }
    // group finishes are recorded only for the groups of batched P2P nodes (several groups on one
    // node), by each such member: a shard contributes the groups of its own batched members
    for (int64_t grp = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; grp < g.G; grp += stride) {
      bool mine = false;
      for (int32_t j = g.grp_ptr[grp]; j < g.grp_ptr[grp + 1] && j < g.grp_ptr[grp] + 2; ++j) {
        const int32_t mn = g.grp_mem[j];
        mine |= g.node_gptr[mn + 1] - g.node_gptr[mn] > 1 && owns_rank(g, g.node_rank[mn], sh);
      }
      if (!mine) continue;
      const int64_t v = gf[grp * Sp + k];
      for (int m = 0; m < L.n; ++m) ((int64_t *)(L.base[m] + L.o_ggcol))[grp] = v;
    }
  }
  __threadfence_system();
}

// Cross-process gather completion: publish flag[self] = epoch at every shard (release, system
// scope; the gather kernel before it on the stream has completed its peer stores) and wait for
// every shard's flag (acquire), with the device watchdog.
__global__ void gather_sync_kernel(ShardLink L, uint32_t epoch, uint32_t *status, uint64_t watchdog_ns) {
  __threadfence_system();
  if (threadIdx.x < L.n) {
    uint32_t *f = (uint32_t *)(L.base[threadIdx.x] + L.o_gflag) + L.self;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
  }
  __syncthreads();
  if (threadIdx.x < L.n) {
    const uint32_t *f = (const uint32_t *)(L.base[L.self] + L.o_gflag) + threadIdx.x;
    uint64_t t0 = 0;
    uint32_t spins = 0;
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if ((int32_t)(v - epoch) >= 0) break;
      __nanosleep(200);
      if ((++spins & 255) == 0) {
        uint64_t now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        if (now - t0 > watchdog_ns) {
          atomicCAS(status, 0u, (uint32_t)PRISM_E_DEADLOCK);
          break;
        }
      }
    }
  }
}

// prism_query_rank: start/finish of one rank's ops in one scenario from fin/gfin (fin layout:
// graph.h fin_off; a sharded replay keeps only its own ranks' rows).
// Start time of node i (rank r, first node rb) in scenario k of a recorded replay: a compute span
// starts its perturbed duration before its finish; a node with one sync group spans exactly the
// group occurrence; a batched P2P node starts at the max over its groups of (group finish - dur').
__device__ __forceinline__ int64_t node_start(const DevGraph &g, const ScenParams &p, int32_t Sp,
                                              const int64_t *fin, const int64_t *gfin, int32_t r, int32_t rb,
                                              int32_t i, int32_t k) {
  const int32_t h0 = g.node_gptr[i], h1 = g.node_gptr[i + 1];
  const int32_t kg = p.first + k;  // global scenario index (perturbation key)
  if (h0 == h1) {  // compute span: exact, finish = start + d'
    int64_t d = nd_dur(g, i);
    if ((p.mask & 1u) && p.amp > 0 && kg > 0)
      d = perturb_x(d, p.seed ^ ((uint64_t)kg * K_GOLD) ^ ((((uint64_t)r << 32) | (uint32_t)(i - rb)) * K_MIX), p);
    return fin[fin_off(g, fin_row(g, i), k, Sp)] - d;
  }
  if (h1 - h0 == 1) {
    const int64_t grp = g.node_grp[h0];
    const uint32_t gbit = (g.grp_uid[grp] >> 56) == PRISM_ROLE_P2P ? 4u : 2u;
    int64_t d = g.grp_dur[grp];
    if ((p.mask & gbit) && p.amp > 0 && kg > 0) d = perturb_x(d, p.seed ^ ((uint64_t)kg * K_GOLD) ^ (g.grp_uid[grp] * K_MIX), p);
    return fin[fin_off(g, fin_row(g, i), k, Sp)] - d;
  }
  int64_t st = 0;
  for (int32_t h = h0; h < h1; ++h) {
    const int64_t grp = g.node_grp[h];
    const uint32_t gbit = (g.grp_uid[grp] >> 56) == PRISM_ROLE_P2P ? 4u : 2u;
    int64_t d = g.grp_dur[grp];
    if ((p.mask & gbit) && p.amp > 0 && kg > 0) d = perturb_x(d, p.seed ^ ((uint64_t)kg * K_GOLD) ^ (g.grp_uid[grp] * K_MIX), p);
    st = max(st, gfin[grp * Sp + k] - d);
  }
  return st;
}

__global__ void query_kernel(DevGraph g, ScenParams p, int32_t Sp, const int64_t *__restrict__ fin,
                             const int64_t *__restrict__ gfin, int32_t r, int32_t k,
                             int64_t *__restrict__ start_out, int64_t *__restrict__ finish_out) {
  const int32_t rb = g.rank_ptr[r], re = g.rank_ptr[r + 1];
  for (int32_t i = rb + blockIdx.x * blockDim.x + threadIdx.x; i < re; i += gridDim.x * blockDim.x) {
    start_out[i - rb] = node_start(g, p, Sp, fin, gfin, r, rb, i, k);
    finish_out[i - rb] = fin[fin_off(g, fin_row(g, i), k, Sp)];
  }
}

// Row a9 in time order (row f2, multi-stream ranks; P:1578 max_memory_allocated): one block per
// rank; the rank's events (+alloc at start: index 2i, -free at finish: 2i+1) are sorted by
// (time, index) — the full 64-bit time, the index as the tie-break — with a bitonic sort in shared
// memory, and prefix-summed; peak = static + max(0, max running total). A running total below
// zero sets PRISM_E_NEGATIVE_MEMORY.
__global__ void __launch_bounds__(1024) peak_time_kernel(DevGraph g, ScenParams p, int32_t Sp,
                                                         const int64_t *__restrict__ fin,
                                                         const int64_t *__restrict__ gfin, int32_t k, int32_t cap,
                                                         int64_t *__restrict__ peak, uint32_t *status) {
  extern __shared__ unsigned long long sm[];
  unsigned long long *key = sm;
  long long *val = (long long *)(sm + cap);
  uint16_t *kix = (uint16_t *)(sm + 2 * (size_t)cap);
  __shared__ long long wsum[32], wmax[32];
  __shared__ int neg;
  for (int32_t r = blockIdx.x; r < g.W; r += gridDim.x) {
    const int32_t rb = g.rank_ptr[r], re = g.rank_ptr[r + 1], len = re - rb;
    for (int32_t x = threadIdx.x; x < cap; x += blockDim.x) {
      const int32_t i = x >> 1;
      if (i < len) {
        const int32_t n = rb + i;
        const bool fr = x & 1;
        const int64_t tm = fr ? fin[fin_off(g, fin_row(g, n), k, Sp)] : node_start(g, p, Sp, fin, gfin, r, rb, n, k);
        key[x] = (unsigned long long)tm;
        kix[x] = (uint16_t)x;
        val[x] = fr ? -nd_free(g, n) : nd_alloc(g, n);
      } else {
        key[x] = ~0ull;
        kix[x] = 0xFFFF;
        val[x] = 0;
      }
    }
    __syncthreads();
    for (int32_t size = 2; size <= cap; size <<= 1)  // bitonic sort, ascending
      for (int32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (int32_t x = threadIdx.x; x < cap; x += blockDim.x) {
          const int32_t y = x ^ stride;
          if (y > x) {
            const bool up = (x & size) == 0;
            const bool gt = key[x] > key[y] || (key[x] == key[y] && kix[x] > kix[y]);
            if (gt == up) {
              const unsigned long long tk = key[x];
              key[x] = key[y];
              key[y] = tk;
              const uint16_t ti = kix[x];
              kix[x] = kix[y];
              kix[y] = ti;
              const long long tv = val[x];
              val[x] = val[y];
              val[y] = tv;
            }
          }
        }
        __syncthreads();
      }
    // running total in sorted order: per-thread chunk sums, block scan of the chunks
    const int32_t per = (cap + (int32_t)blockDim.x - 1) / (int32_t)blockDim.x;
    const int32_t x0 = threadIdx.x * per;
    long long s = 0, mx = 0;
    for (int32_t x = x0; x < x0 + per && x < cap; ++x) {
      s += val[x];
      mx = max(mx, s);
    }
    // exclusive prefix of chunk sums (warp shuffles + per-warp totals)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long incl = s;
    for (int off = 1; off < 32; off <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    if (threadIdx.x == 0) neg = 0;
    __syncthreads();
    long long woff = 0;
    for (int w = 0; w < wid; ++w) woff += wsum[w];
    const long long before = woff + incl - s;
    long long run = before, best = 0, low = 0;
    for (int32_t x = x0; x < x0 + per && x < cap; ++x) {
      run += val[x];
      best = max(best, run);
      low = min(low, run);
    }
    (void)mx;
    if (low < 0) neg = 1;
    for (int off = 16; off; off >>= 1) best = max(best, (long long)__shfl_xor_sync(0xffffffffu, best, off));
    if (lane == 0) wmax[wid] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long b = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b = max(b, wmax[w]);
      peak[r] = g.static_mem[g.rank_stage[r]] + b;
      if (neg) atomicCAS(status, 0u, (uint32_t)PRISM_E_NEGATIVE_MEMORY);
    }
    __syncthreads();
  }
}

template <int L, int SPL>
cudaError_t level_t(const DevGraph &g, const ScenParams &p, const Tile *tiles, int32_t ntiles,
                    int32_t max_cnt, int64_t *fin, int64_t *gfin, int nchunks, cudaStream_t st) {
  const size_t smem = (size_t)max_cnt * L * SPL * sizeof(unsigned long long);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(level_kernel<L, SPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(ntiles, nchunks);
  level_kernel<L, SPL><<<grid, 256, smem, st>>>(g, p, tiles, fin, gfin);
  return cudaGetLastError();
}

template <int L, int SPL>
cudaError_t tail_t(const DevGraph &g, const ScenParams &p, int64_t *fin, const int64_t *gfin,
                   int64_t *rank_end, int nchunks, cudaStream_t st) {
  constexpr int TEAMS = 256 / L;
  int blocks = (g.W + TEAMS - 1) / TEAMS;
  if (blocks < 1) blocks = 1;
  dim3 grid(blocks, nchunks);
  tail_kernel<L, SPL><<<grid, 256, 0, st>>>(g, p, fin, gfin, rank_end);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_level(const DevGraph &g, const ScenParams &p, const Tile *tiles, int32_t ntiles,
                         int32_t max_cnt, int64_t *fin, int64_t *gfin, int lanes, int nchunks,
                         cudaStream_t st) {
  switch (lanes) {
    case 1: return level_t<1, 1>(g, p, tiles, ntiles, max_cnt, fin, gfin, nchunks, st);
    case 2: return level_t<2, 1>(g, p, tiles, ntiles, max_cnt, fin, gfin, nchunks, st);
    case 4: return level_t<4, 1>(g, p, tiles, ntiles, max_cnt, fin, gfin, nchunks, st);
    case 8: return level_t<8, 1>(g, p, tiles, ntiles, max_cnt, fin, gfin, nchunks, st);
    case 16: return level_t<16, 1>(g, p, tiles, ntiles, max_cnt, fin, gfin, nchunks, st);
    default: return level_t<32, 2>(g, p, tiles, ntiles, max_cnt, fin, gfin, nchunks, st);
  }
}

cudaError_t launch_tail(const DevGraph &g, const ScenParams &p, int64_t *fin, const int64_t *gfin,
                        int64_t *rank_end, int lanes, int nchunks, cudaStream_t st) {
  switch (lanes) {
    case 1: return tail_t<1, 1>(g, p, fin, gfin, rank_end, nchunks, st);
    case 2: return tail_t<2, 1>(g, p, fin, gfin, rank_end, nchunks, st);
    case 4: return tail_t<4, 1>(g, p, fin, gfin, rank_end, nchunks, st);
    case 8: return tail_t<8, 1>(g, p, fin, gfin, rank_end, nchunks, st);
    case 16: return tail_t<16, 1>(g, p, fin, gfin, rank_end, nchunks, st);
    default: return tail_t<32, 2>(g, p, fin, gfin, rank_end, nchunks, st);
  }
}

// One block: word 0 = abort status of the previous waiting replay, word 1 = sticky first error
// (reported and cleared by the host at its next synchronising call). Reading word 0, folding it
// and clearing it happen in one block (ordered by __syncthreads), before this replay's kernel.
__global__ void __launch_bounds__(1024) replay_guard_kernel(uint32_t *words, int64_t *rslot, size_t rslot_words,
                                                           int64_t *rres, size_t rres_words, int64_t fill) {
  __shared__ uint32_t s;
  if (threadIdx.x == 0) s = words[0];
  __syncthreads();
  if (s == 0) return;
  if (rslot) {
    for (size_t i = threadIdx.x; i < rslot_words; i += blockDim.x) rslot[i] = fill;
    for (size_t i = threadIdx.x; i < rres_words; i += blockDim.x) rres[i] = fill;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (words[1] == 0) words[1] = s;
    words[0] = 0;
  }
}

cudaError_t launch_replay_guard(uint32_t *words, int64_t *rslot, size_t rslot_words, int64_t *rres, size_t rres_words,
                                int parity, cudaStream_t st) {
  // "not yet" under the replay's parity: slots hold t (parity 0) or ~t (parity 1), valid when the
  // decoded value is >= 0, so -1 reads "not yet" under parity 0 and 0 (~0 = -1) under parity 1
  replay_guard_kernel<<<1, 1024, 0, st>>>(words, rslot, rslot_words, rres, rres_words, parity ? 0 : -1);
  return cudaGetLastError();
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

cudaError_t launch_reduce(int32_t W, int32_t S, int32_t Sp, const int64_t *rank_end, int64_t *iter,
                          cudaStream_t st) {
  if (S <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(iter, 0, (size_t)S * 8, st);
  if (e != cudaSuccess) return e;
  const int ry = std::max(1, std::min(64, (W + 7) / 8));
  reduce_iter_kernel<<<dim3((S + 31) / 32, ry), 256, 0, st>>>(W, S, Sp, rank_end, iter);
  return cudaGetLastError();
}

// With lazy module loading (CUDA 12 default) the first launch of a kernel loads it, and loading
// waits for the work already running on the device; a sharded replay launches its reduce kernels
// while its cell kernel is still waiting for peers, so every kernel that can be launched behind a
// running replay is loaded up front (prism_build_graph calls this once per device).
cudaError_t preload_replay_kernels() {
  cudaFuncAttributes a;
  const void *fns[] = {(const void *)reduce_iter_kernel, (const void *)shard_partial_kernel,
                       (const void *)shard_exchange_kernel, (const void *)query_kernel,
                       (const void *)peak_time_kernel, (const void *)replay_guard_kernel,
                       (const void *)local_group_reduce_kernel, (const void *)gather_kernel,
                       (const void *)gather_sync_kernel};
  for (const void *f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_gather(const DevGraph &g, const ShardLink &link, const int64_t *fin, const int64_t *gfin,
                          int32_t Sp, int32_t k, uint32_t epoch, uint32_t *status, cudaStream_t st) {
  gather_kernel<<<num_sms() * 8, 256, 0, st>>>(g, link, fin, gfin, Sp, k);
  if (link.lg == 0) gather_sync_kernel<<<1, 32, 0, st>>>(link, epoch, status, g.watchdog_ns);
  return cudaGetLastError();
}

cudaError_t launch_local_group_reduce(const DevGraph &g, const ShardLink &link, int32_t S, int32_t Sp,
                                      int64_t *iter, cudaStream_t st) {
  local_group_reduce_kernel<<<S, 256, 0, st>>>(g, link, Sp, iter);
  return cudaGetLastError();
}

cudaError_t launch_shard_reduce(const DevGraph &g, const ShardLink &link, int32_t S, int32_t Sp,
                                const int64_t *rank_end, int64_t *part_local, int64_t *iter,
                                uint32_t *status, cudaStream_t st) {
  shard_partial_kernel<<<S, 256, 0, st>>>(g, Sp, rank_end, part_local);
  shard_exchange_kernel<<<1, 1024, 0, st>>>(link, S, Sp, part_local, iter, status, g.watchdog_ns);
  return cudaGetLastError();
}

cudaError_t launch_peak_time(const DevGraph &g, const ScenParams &p, int32_t Sp, const int64_t *fin,
                             const int64_t *gfin, int32_t k, int32_t max_len, int64_t *peak, uint32_t *status,
                             cudaStream_t st) {
  int32_t cap = 2;
  while (cap < 2 * max_len) cap <<= 1;
  const size_t smem = (size_t)cap * 18;
  cudaError_t e = cudaFuncSetAttribute(peak_time_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int threads = cap >= 1024 ? 1024 : (cap < 32 ? 32 : cap);  // whole warps (shuffle scans)
  peak_time_kernel<<<g.W < num_sms() * 2 ? g.W : num_sms() * 2, threads, smem, st>>>(g, p, Sp, fin, gfin, k, cap, peak, status);
  return cudaGetLastError();
}

cudaError_t launch_query(const DevGraph &g, const ScenParams &p, int32_t Sp, const int64_t *fin,
                         const int64_t *gfin, int32_t rank, int32_t scen,
                         int64_t *start_out, int64_t *finish_out, cudaStream_t st) {
  query_kernel<<<64, 256, 0, st>>>(g, p, Sp, fin, gfin, rank, scen, start_out, finish_out);
  return cudaGetLastError();
}

}  // namespace prism
