// replay_ranks.cu — the single-scenario replay (rows a6-a8 at S = 1): lane = rank.
//
// Same semantics as the cell kernel (readings Z2-Z5), laid out
// for ONE scenario: with lane = scenario, an S = 1 replay would leave 31 lanes idle while one
// lane hashes all tp ranks of its cell op after op; here a warp owns 32 ranks of one pipeline
// stage (tp_i fastest, then dp_i; they all run the stage template), one per lane, so an op
// costs each lane one perturbation and the dependency chain through the pipeline advances ~tp
// times faster. Per op:
//   compute span      : t += dur'(own rank)
//   TP collective     : segmented max over the tp lanes of the lane's TP group (xor shuffles,
//                       tp a power of two) + the group's dur'
//   chained collective: t += dur'(own group) (every member sits at the previous occurrence's
//                       shared finish, reading of plan.cpp)
//   cross-warp group  : the lane deposits its ready time into its own ready slot (value-as-flag,
//                       parity-encoded; a large group: red.max + acq_rel arrival, the completing
//                       member publishes the max in a result slot) and polls its partners;
//                       the node finishes at the max over its groups (start + dur').
// Template records (class, duration, group type / occurrence) are broadcast to the lanes from a
// 32-op batch loaded one batch ahead; per-rank durations (prism_set_durations) are read per lane
// one op ahead. Every warp of the launch is co-resident (cooperative launch) and a %globaltimer
// watchdog turns any stall into PRISM_E_DEADLOCK.
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
  const int64_t pm = a.parity ? -1 : 0;
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
  uint32_t spins_total = 0;
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
        const int32_t h0 = active ? g.node_gptr[rb + i] : 0;
        const int32_t ns = active ? g.node_gptr[rb + i + 1] - h0 : 0;
        uint32_t meta[kMaxSlots];
        int32_t hb[kMaxSlots];
        int64_t val[kMaxSlots];
        uint32_t pend = 0;
#pragma unroll
        for (int q = 0; q < kMaxSlots; ++q) {
          meta[q] = 0;
          hb[q] = 0;
          val[q] = t;
          if (q < ns) {
            meta[q] = g.h_meta[h0 + q];
            hb[q] = g.h_base[h0 + q];
            pend |= 1u << q;
            if (!(meta[q] & 0x80000000u)) {
              str64(a.rslot + hb[q] + (int32_t)((meta[q] >> 16) & 0x7FFF), t ^ pm);
            } else {  // large group: accumulate, arrive; the completing member publishes the max
              asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(a.acc + hb[q]), "l"((uint64_t)t) : "memory");
              uint32_t old;
              asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.arrive + hb[q]) : "memory");
              if (old + 1 == (meta[q] & 0xFFFF)) {
                val[q] = ldr64(a.acc + hb[q]);
                str64(a.rres + hb[q], val[q] ^ pm);
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
            if (meta[q] & 0x80000000u) {
              const int64_t v = ldr64(a.rres + hb[q]) ^ pm;
              ok = v >= 0;
              m = max(m, v);
            } else {
              const int32_t size = (int32_t)(meta[q] & 0xFFFF), own = (int32_t)((meta[q] >> 16) & 0x7FFF);
              for (int32_t mm = 0; mm < size; ++mm) {
                if (mm == own) continue;
                const int64_t v = ldr64(a.rslot + hb[q] + mm) ^ pm;
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
          ++spins_total;
          if (spins > 2) __nanosleep(min(1024u, 32u << min(spins, 10u)));
          if ((spins & 63) == 0) {
            if (ldr32(a.status) != 0) return;
            if (t0 == 0) t0 = gtimer();
            if (gtimer() - t0 > a.timeout_ns) {
              atomicCAS(a.status, 0u, (uint32_t)PRISM_E_DEADLOCK);
              return;
            }
          }
        }
        int64_t fr = 0;
#pragma unroll
        for (int q = 0; q < kMaxSlots; ++q) {
          if (q >= ns) continue;
          const int32_t h = h0 + q;
          int64_t gd = g.h_dur[h];
          const uint64_t uid = g.h_uid[h];
          const bool pr = (uid >> 56) == PRISM_ROLE_P2P ? ppert : gpert;
          if (pr) gd = perturb_x(gd, sx ^ (uid * K_MIX), p);
          const int64_t f = val[q] + gd;
          fr = max(fr, f);
          if (ns > 1) gfin[g.node_grp[h]] = f;  // batched P2P groups' finishes, for queries
        }
        if (active) t = fr;
      }
      if (p.record && active) fin[frow0 + (int64_t)i * fstride] = t;
    }
  }
  if (active) rank_end[r] = t;
  (void)rs;
  (void)spins_total;
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
  if (blocks) *blocks = (int)need;
  return need >= 1 && (int64_t)per_sm * sms >= need;
}

cudaError_t preload_rank_kernels() {
  cudaFuncAttributes at;
  cudaError_t e = cudaFuncGetAttributes(&at, (const void *)rank_kernel<false>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&at, (const void *)rank_kernel<true>);
  return e;
}

cudaError_t launch_ranks(const DevGraph &g, const ScenParams &p, int64_t *rslot, int64_t *acc, int64_t *rres,
                         uint32_t *arrive, uint32_t *status, int parity, int64_t *fin, int64_t *gfin,
                         int64_t *rank_end, cudaStream_t st) {
  int blocks = 0;
  if (!ranks_fit(g, &blocks)) return cudaErrorCooperativeLaunchTooLarge;
  const int32_t per_warp_dp = 32 / g.tp;
  RankArgs a{rslot, acc, rres, arrive, status, g.watchdog_ns, parity, per_warp_dp,
             (int32_t)((g.dp + per_warp_dp - 1) / per_warp_dp)};
  DevGraph gg = g;
  ScenParams pp = p;
  void *args[] = {&gg, &pp, &a, &fin, &gfin, &rank_end};
  const void *fn = g.per_rank_dur ? (const void *)rank_kernel<true> : (const void *)rank_kernel<false>;
  return cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(32), args, 0, st);
}

}  // namespace prism
