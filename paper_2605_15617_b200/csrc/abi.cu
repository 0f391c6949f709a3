// abi.cu — the C ABI (include/prism.h): graph handles, device memory, launch orchestration.
//
// prism_build_graph = host validation + quotient plan (plan.cpp) -> H2D of the per-stage tables
// (KBs) -> expand kernels (rows a1-a4) on the caller's stream. prism_replay = one level_kernel
// launch per frontier level (rows a5-a7), then tail + reduce (a8). prism_peak_memory = peak_kernel
// (a9). No CPU fallback: every compute entry point fails with PRISM_E_CUDA without a device.
#include <cuda_runtime.h>

#include <malloc.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "graph.h"

using namespace prism;

namespace {

thread_local std::string t_err;

// Pinned host status slots (4 words per graph: [0] abort status of the last waiting replay, [1]
// sticky first abort of earlier replays, [2] time-ordered memory scan status), shared by all graphs
// (cudaHostAlloc / cudaFreeHost per graph would synchronize the device on every build/destroy).
std::mutex g_pin_mu;
uint32_t *g_pin = nullptr;
std::vector<int> g_pin_free;
constexpr int kPinWords = 4096;
constexpr int kPinSlot = 4;  // words per graph
// A word whose graph was destroyed is reclaimed once the event recorded behind its last status
// copy has completed (a host callback on the stream would stall the stream's next kernels until
// the host ran it: a bubble in every bench step).
struct PinPending {
  int idx;
  cudaEvent_t ev;
  int dev;
};
std::vector<PinPending> g_pin_pending;
std::vector<PinPending> g_pin_events;  // completed events for reuse (idx unused)
void pin_reclaim_locked() {
  for (size_t i = 0; i < g_pin_pending.size();) {
    PinPending &q = g_pin_pending[i];
    if (cudaEventQuery(q.ev) == cudaSuccess) {
      g_pin_free.push_back(q.idx);
      g_pin_events.push_back(q);
      q = g_pin_pending.back();
      g_pin_pending.pop_back();
    } else {
      ++i;
    }
  }
}
uint32_t *pin_take() {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  if (!g_pin) {
    if (cudaHostAlloc((void **)&g_pin, kPinWords * 4, cudaHostAllocDefault) != cudaSuccess) {
      g_pin = nullptr;
      return nullptr;
    }
    for (int i = kPinWords - kPinSlot; i >= 0; i -= kPinSlot) g_pin_free.push_back(i);
  }
  if (g_pin_free.empty()) {
    pin_reclaim_locked();
    cudaGetLastError();  // cudaErrorNotReady of the queries is not an error
  }
  if (g_pin_free.empty()) return nullptr;
  const int i = g_pin_free.back();
  g_pin_free.pop_back();
  for (int j = 0; j < kPinSlot; ++j) g_pin[i + j] = 0;
  return g_pin + i;
}
// Returns word p once the work queued so far on stream st (device dev) has completed.
void pin_give_after(uint32_t *p, cudaStream_t st, int dev) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  const int idx = (int)(p - g_pin);
  cudaEvent_t ev = nullptr;
  for (size_t i = 0; i < g_pin_events.size(); ++i)
    if (g_pin_events[i].dev == dev) {
      ev = g_pin_events[i].ev;
      g_pin_events[i] = g_pin_events.back();
      g_pin_events.pop_back();
      break;
    }
  if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) ev = nullptr;
  if (ev && cudaEventRecord(ev, st) == cudaSuccess) {
    g_pin_pending.push_back(PinPending{idx, ev, dev});
    return;
  }
  cudaGetLastError();
  cudaStreamSynchronize(st);
  g_pin_free.push_back(idx);
  if (ev) g_pin_events.push_back(PinPending{-1, ev, dev});
}
std::mutex g_alloc_mu;
prism_alloc_fn g_alloc = nullptr;
prism_free_fn g_free = nullptr;
void *g_alloc_ctx = nullptr;

// PRISM_TRACE=1: host timestamps of the launch sequence (diagnostics of blocking API calls).
void trace(const char *what) {
  static const bool on = std::getenv("PRISM_TRACE") != nullptr;
  if (!on) return;
  static const auto t0 = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[prism %9.3f ms] %s\n",
               std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), what);
}

prism_status fail(prism_status s, const std::string &m) {
  t_err = m;
  return s;
}

#define CU(call)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(e_ == cudaErrorMemoryAllocation ? PRISM_E_OOM : PRISM_E_CUDA,              \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                       \
  } while (0)

}  // namespace

namespace {
// The host plan allocates a few MB of short-lived tables per build; with glibc's default mmap
// threshold every build page-faults them in afresh (~0.9 ms of a ~2.3 ms plan for C5). Keep
// such blocks in the heap so repeated builds reuse warm pages.
struct MallocTuning {
  MallocTuning() {
    mallopt(M_MMAP_THRESHOLD, 64 << 20);
    mallopt(M_TRIM_THRESHOLD, 256 << 20);
  }
} g_malloc_tuning;

// Pinned staging buffers of the build uploads. From pageable memory cudaMemcpyAsync returns only
// after the copy engine has taken the data — i.e. after every earlier operation on the stream (the
// previous step's replay) — so the host could not plan the next graph while the device replays;
// from pinned memory the upload is queued and the host runs ahead. A small process-wide ring of
// buffers; a slot is reused once the event recorded after its copy has completed.
struct PinnedRing {
  struct Slot {
    unsigned char *p = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    int dev = -1;
  };
  std::mutex mu;
  Slot slot[4];
  int next = 0;
};
PinnedRing &pinned_ring() {
  static PinnedRing *r = new PinnedRing;  // never destroyed: the buffers live for the process
  return *r;
}
struct PinnedStage {
  unsigned char *ptr = nullptr;
  int idx = -1;
  explicit PinnedStage(size_t bytes) {
    PinnedRing &R = pinned_ring();
    std::lock_guard<std::mutex> lk(R.mu);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    const int i = R.next;
    PinnedRing::Slot &S = R.slot[i];
    if (S.ev) {
      cudaEventSynchronize(S.ev);  // the slot's previous copy has completed
      if (S.dev != dev) {
        cudaEventDestroy(S.ev);
        S.ev = nullptr;
      }
    }
    if (!S.ev) {
      if (cudaEventCreateWithFlags(&S.ev, cudaEventDisableTiming) != cudaSuccess) {
        S.ev = nullptr;
        cudaGetLastError();
        return;
      }
      S.dev = dev;
    }
    if (S.cap < bytes) {
      // every slot is (re)allocated at once, at the size this build needs: pinning host memory
      // (cudaMallocHost) takes tens of milliseconds, and a slot first used by a later build stalled
      // that build's host thread (a serving loop's 4th build: one 47 ms stall in a timed region)
      const size_t cap = std::max(bytes + bytes / 4, (size_t)1 << 20);
      for (int k = 0; k < 4; ++k) {
        PinnedRing::Slot &T = R.slot[(i + k) % 4];
        if (T.cap >= bytes) continue;
        if (T.ev && k > 0) cudaEventSynchronize(T.ev);  // its previous copy has completed
        if (T.p) cudaFreeHost(T.p);
        T.p = nullptr;
        T.cap = 0;
        if (cudaMallocHost((void **)&T.p, cap) != cudaSuccess) {
          T.p = nullptr;
          cudaGetLastError();
          if (k == 0) return;
          continue;
        }
        T.cap = cap;
      }
    }
    R.next = (i + 1) % 4;
    idx = i;
    ptr = S.p;
  }
  // records the completion event of the copy just queued on `st`; the slot is not handed out
  // again before that event has completed
  void release(cudaStream_t st) {
    if (idx < 0) return;
    PinnedRing &R = pinned_ring();
    std::lock_guard<std::mutex> lk(R.mu);
    cudaEventRecord(R.slot[idx].ev, st);
  }
};
}  // namespace

struct prism_graph_s {
  Plan plan;
  DevGraph dg{};
  cudaStream_t stream = nullptr;
  int device = 0;
  prism_alloc_fn alloc = nullptr;
  prism_free_fn free_fn = nullptr;
  void *ctx = nullptr;
  std::vector<std::pair<void *, size_t>> blocks;  // structure allocations
  int64_t structure_bytes = 0;
  // replay state: the arrays below live in ONE device block (`state`, carved per replay), so a
  // replay allocates at most once through the allocator hooks (each hook call costs the Python
  // binding tens of microseconds of host time on the bench step's critical path)
  unsigned char *state = nullptr;
  size_t state_cap = 0;
  size_t state_off[8] = {}, state_len[8] = {};  // the current carve (offsets, bytes)
  int64_t *fin = nullptr;
  size_t fin_bytes = 0;
  int64_t *gfin = nullptr;
  size_t gfin_bytes = 0;
  int64_t *rank_end = nullptr;
  size_t rank_end_bytes = 0;
  int64_t *iter = nullptr;
  size_t iter_bytes = 0;
  int64_t *scratch = nullptr;
  size_t scratch_bytes = 0;
  // cell-kernel state
  int64_t *rslot = nullptr;   // ready slots; parity-encoded, see replay_cells.cu
  size_t rslot_bytes = 0;
  int parity = 0;             // encoding of the next replay
  bool rslot_dirty = true;    // needs a reset (new allocation / aborted replay / new stride)
  int32_t rslot_Sp = 0;
  int64_t *acc = nullptr;     // large-group accumulators [G_large][Sp]
  size_t acc_bytes = 0;
  int64_t *rres = nullptr;    // large-group result slots [G_large][Sp] (parity-encoded)
  size_t rres_bytes = 0;
  uint32_t *sync_words = nullptr;  // arrive[G_large x chunks] (sharded: unused)
  size_t sync_bytes = 0;
  uint32_t *words = nullptr;       // device: [0] replay abort status, [1] sticky abort, [2] memory
                                   // scan status (part of the structure allocation, zeroed at build)
  uint32_t *h_status = nullptr;    // pinned copy of words[0..2] (slot of kPinSlot words)
  int last_algo = 0;
  int recorded = 0;
  // fin keeps rows [fin_node0, fin_node0 + fin_rows) (all nodes unless sharded)
  int64_t fin_node0 = 0, fin_rows = 0;
  // row e: sharding (n_shards > 1)
  int n_shards = 1, shard = 0;
  unsigned char *ex = nullptr;          // exchange buffer (cudaMalloc: IPC-exportable)
  size_t ex_bytes = 0;
  int32_t ex_S = 0, ex_Sp = 0;
  ShardLink link{};
  bool connected = false;
  bool local_group = false;
  uint32_t gather_epoch = 0;            // prism_shard_gather calls since prepare
  int32_t gathered_k = -1;              // scenario held in the gather columns (-1: none)             // connected to peers on this same device: such shards can
                                        // only replay together (prism_replay_local_shards)
  std::vector<void *> ipc_open;         // peer buffers opened with cudaIpcOpenMemHandle
  int64_t *part = nullptr;              // [S] local partial iteration times
  size_t part_bytes = 0;
  ScenParams last{};
  int32_t last_Sp = 0;
  // tile plan cache (depends on lanes)
  int tiles_lanes = -1;
  Tile *tiles = nullptr;
  size_t tiles_bytes = 0;
  std::vector<int32_t> lvl_tile_ptr, lvl_max_cnt;
  int64_t launches = 0;
  bool oom = false;
  std::vector<unsigned char> staging;  // packed host tables of the build upload
  std::vector<uint32_t> tmpl_labels;     // template labels (label-override validation)
  // profiling events: 0/1 expand, 2/3 levels, 4 tail end, 5 reduce end, 6/7 peak
  bool profile = false;
  cudaEvent_t ev[8] = {};
  bool ev_done[8] = {};
  void rec(int i) {
    if (profile) {
      cudaEventRecord(ev[i], stream);
      ev_done[i] = true;
    }
  }

  // rows f1/f3/f4: per-node duration / memory overrides. The inputs of prism_set_durations (din)
  // and prism_set_moe_load (moe) are kept on the device; the derived arrays (ov) are recomputed
  // from both whenever either changes, and the replay reads them through dov's pointers.
  bool ov_active = false;
  DevGraph dov{};
  unsigned char *ov = nullptr;
  DurIn din{};
  bool din_any = false;
  unsigned char *din_blk = nullptr;
  MoeIn moe{};
  unsigned char *moe_blk = nullptr;
  const DevGraph &cur() const { return ov_active ? dov : dg; }
  // critical-path scratch
  int32_t *crit = nullptr;
  size_t crit_bytes = 0;

  void *dalloc(size_t bytes) {
    if (bytes == 0) bytes = 16;
    void *p = nullptr;
    if (alloc) {
      p = alloc(bytes, (void *)stream, ctx);
    } else if (cudaMallocAsync(&p, bytes, stream) != cudaSuccess) {
      p = nullptr;
    }
    return p;
  }
  void dfree(void *p) {
    if (!p) return;
    if (free_fn) free_fn(p, (void *)stream, ctx);
    else cudaFreeAsync(p, stream);
  }
  template <class T>
  T *take(size_t count) {  // structure allocation, freed with the graph
    size_t b = count * sizeof(T);
    void *p = dalloc(b);
    if (p) {
      blocks.emplace_back(p, b);
      structure_bytes += (int64_t)b;
    } else {
      oom = true;
    }
    return (T *)p;
  }
  template <class T>
  bool ensure(T *&p, size_t &cap, size_t bytes) {
    if (cap >= bytes && p) return true;
    dfree(p);
    p = (T *)dalloc(bytes);
    cap = p ? bytes : 0;
    return p != nullptr;
  }
  ~prism_graph_s() {
    trace("destroy: begin");
    dfree(state);
    dfree(iter);
    dfree(scratch);
    dfree(tiles);
    dfree(ov);
    dfree(din_blk);
    dfree(moe_blk);
    dfree(crit);
    trace("destroy: buffers freed");
    if (h_status) {  // returned to the pool once the stream has passed its pending status copy
      int cur = -1;
      cudaGetDevice(&cur);
      if (device >= 0 && cur != device) cudaSetDevice(device);
      pin_give_after(h_status, stream, device);
      if (device >= 0 && cur >= 0 && cur != device) cudaSetDevice(cur);
    }
    trace("destroy: status slot returned");
    for (auto &b : blocks) dfree(b.first);  // stream-ordered frees: no host wait needed
    trace("destroy: structure freed");
    if (ex || !ipc_open.empty()) {  // the exchange buffer is not stream-ordered memory
      cudaStreamSynchronize(stream);
      for (void *p : ipc_open) cudaIpcCloseMemHandle(p);
      if (ex) cudaFree(ex);
    }
    for (auto &e : ev)
      if (e) cudaEventDestroy(e);
  }
};

extern "C" {

const char *prism_status_string(prism_status s) {
  switch (s) {
    case PRISM_OK: return "PRISM_OK";
    case PRISM_E_INVALID_ARG: return "PRISM_E_INVALID_ARG";
    case PRISM_E_INVALID_SPEC: return "PRISM_E_INVALID_SPEC";
    case PRISM_E_GA_TOO_SMALL: return "PRISM_E_GA_TOO_SMALL";
    case PRISM_E_TEMPLATE_MISMATCH: return "PRISM_E_TEMPLATE_MISMATCH";
    case PRISM_E_DEADLOCK: return "PRISM_E_DEADLOCK";
    case PRISM_E_NEGATIVE_MEMORY: return "PRISM_E_NEGATIVE_MEMORY";
    case PRISM_E_UNKNOWN_RANK: return "PRISM_E_UNKNOWN_RANK";
    case PRISM_E_UNKNOWN_LABEL: return "PRISM_E_UNKNOWN_LABEL";
    case PRISM_E_NOT_REPLAYED: return "PRISM_E_NOT_REPLAYED";
    case PRISM_E_OOM: return "PRISM_E_OOM";
    case PRISM_E_CUDA: return "PRISM_E_CUDA";
    case PRISM_E_NCCL: return "PRISM_E_NCCL";
    default: return "PRISM_E_UNKNOWN_STATUS";
  }
}

const char *prism_last_error(void) { return t_err.c_str(); }

int32_t prism_abi_version(void) { return PRISM_ABI_VERSION; }

prism_status prism_set_allocator(prism_alloc_fn alloc, prism_free_fn free_fn, void *ctx) {
  if ((alloc == nullptr) != (free_fn == nullptr)) return fail(PRISM_E_INVALID_ARG, "alloc and free hooks must be set together");
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  g_alloc = alloc;
  g_free = free_fn;
  g_alloc_ctx = ctx;
  return PRISM_OK;
}

}  // extern "C"

namespace {
// Row e, SURVEY §8.4 planner: the shard axis whose blocks cut the fewest exchanged synchronisations. DP blocks
// (shard of a rank = dp_i / (dp/n)) keep TP groups and P2P messages local and cut DP and WORLD
// collectives, EP all-to-alls wider than a block and EDP groups; PP-stage blocks keep every
// collective but WORLD local and cut the P2P messages at block edges. opts->flags may force one.
prism_status choose_shard_axis(const Plan &P, int n, int flags, int &axis, std::string &err) {
  const bool dp_ok = P.topo.dp % n == 0, pp_ok = P.topo.pp % n == 0;
  const bool want_dp = flags & PRISM_BUILD_SHARD_DP, want_pp = flags & PRISM_BUILD_SHARD_PP;
  if (want_dp && want_pp) {
    err = "PRISM_BUILD_SHARD_DP and PRISM_BUILD_SHARD_PP are exclusive";
    return PRISM_E_INVALID_ARG;
  }
  if ((want_dp && !dp_ok) || (want_pp && !pp_ok) || (!dp_ok && !pp_ok)) {
    err = "the shard count must divide dp (DP blocks) or pp (PP-stage blocks)";
    return PRISM_E_INVALID_SPEC;
  }
  if (want_dp || !pp_ok) {
    axis = 0;
    return PRISM_OK;
  }
  if (want_pp || !dp_ok) {
    axis = 1;
    return PRISM_OK;
  }
  // cost of an axis = the template-level synchronisations it cuts that the replay must exchange
  // (a chained collective, class 3, resolves locally): each one puts a cross-shard rendezvous on a
  // rank's chain, whatever the number of its instances (they run side by side)
  const int64_t Bd = P.topo.dp / n, Bp = P.topo.pp / n, ep = P.topo.ep;
  int64_t cut_dp = 0, cut_pp = 0;
  for (const QGroup &q : P.q) {
    const int64_t m = (P.t_cls[P.stage_op0[q.stage] + q.tidx] & 0xF) == 3 ? 0 : 1;
    switch (q.type) {
      case PRISM_ROLE_DP: cut_dp += m; break;
      case PRISM_ROLE_WORLD: cut_dp += m; cut_pp += m; break;
      case PRISM_ROLE_EP: if (ep > Bd || Bd % ep != 0) cut_dp += m; break;
      case PRISM_ROLE_EDP: if (q.size > 1) cut_dp += m; break;
      case PRISM_ROLE_P2P: if (q.stage / Bp != q.stage2 / Bp) cut_pp += m; break;
      default: break;
    }
  }
  axis = cut_pp < cut_dp ? 1 : 0;
  return PRISM_OK;
}
// Plan cache (host): a build whose topology, template bytes and shard options equal an earlier
// build's reuses that build's validated plan (plan_graph, the shard axis and the replica-cell
// rewrite: O(template ops), ~1.6 ms for C5) — a serving loop rebuilding one workload then pays a
// byte comparison and a copy. The key is the inputs themselves (exact; no hash), four entries,
// least recently used first out. PRISM_PLAN_CACHE=0 turns it off.
struct PlanCacheEntry {
  std::vector<unsigned char> key;
  Plan plan;
  int axis = 0;
};
std::mutex g_plan_mu;
std::vector<PlanCacheEntry> g_plan_cache;  // most recently used last
constexpr size_t kPlanCacheEntries = 4;

bool plan_key(const prism_topology &t, const prism_templates &tm, int n_shards, int shard, uint32_t flags,
              int env_a, int env_b, std::vector<unsigned char> &key) {
  static const bool off = [] {
    const char *e = std::getenv("PRISM_PLAN_CACHE");
    return e && std::atoi(e) == 0;
  }();
  // only well-formed inputs are keyed (plan_graph reports everything else)
  if (off || t.pp < 1 || t.pp > (1 << 16) || tm.n_ops < 0 || tm.n_ops > (int64_t(1) << 28) ||
      (tm.n_ops > 0 && !tm.ops) || !tm.tmpl_ptr || !tm.static_mem)
    return false;
  const size_t nops = (size_t)tm.n_ops * sizeof(prism_op), nptr = (size_t)(t.pp + 1) * 8, nst = (size_t)t.pp * 8;
  key.resize(sizeof t + 8 + 5 * 4 + nops + nptr + nst);
  unsigned char *k = key.data();
  const int32_t o[5] = {n_shards, shard, (int32_t)flags, env_a, env_b};
  std::memcpy(k, &t, sizeof t);
  k += sizeof t;
  std::memcpy(k, &tm.n_ops, 8);
  k += 8;
  std::memcpy(k, o, sizeof o);
  k += sizeof o;
  if (nops) std::memcpy(k, tm.ops, nops);
  k += nops;
  std::memcpy(k, tm.tmpl_ptr, nptr);
  k += nptr;
  std::memcpy(k, tm.static_mem, nst);
  return true;
}

bool plan_cache_get(const std::vector<unsigned char> &key, Plan &plan, int &axis) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  for (size_t i = g_plan_cache.size(); i-- > 0;) {
    PlanCacheEntry &e = g_plan_cache[i];
    if (e.key.size() == key.size() && std::memcmp(e.key.data(), key.data(), key.size()) == 0) {
      plan = e.plan;
      axis = e.axis;
      if (i + 1 != g_plan_cache.size()) std::rotate(g_plan_cache.begin() + i, g_plan_cache.begin() + i + 1, g_plan_cache.end());
      return true;
    }
  }
  return false;
}

void plan_cache_put(std::vector<unsigned char> &&key, const Plan &plan, int axis) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  if (g_plan_cache.size() >= kPlanCacheEntries) g_plan_cache.erase(g_plan_cache.begin());
  g_plan_cache.push_back(PlanCacheEntry{std::move(key), plan, axis});
}
}  // namespace

extern "C" {

prism_status prism_plan(const prism_topology *topo, const prism_templates *tmpl, int64_t out[8]) {
  if (!topo || !tmpl || !out) return fail(PRISM_E_INVALID_ARG, "null argument");
  trace("build: begin");
  Plan plan;
  std::string err;
  prism_status st = plan_graph(*topo, *tmpl, plan, err);
  if (st != PRISM_OK) return fail(st, err);
  trace("build: planned");
  out[0] = plan.W;
  out[1] = plan.N;
  out[2] = plan.G;
  out[3] = plan.M;
  out[4] = plan.levels;
  out[5] = (int64_t)plan.q.size();
  out[6] = plan.sync_nodes;
  out[7] = plan.max_group;
  return PRISM_OK;
}

prism_status prism_build_graph(const prism_topology *topo, const prism_templates *tmpl,
                               const prism_build_opts *opts, prism_graph_t *out) {
  if (!topo || !tmpl || !out) return fail(PRISM_E_INVALID_ARG, "null argument");
  *out = nullptr;
  const int n_shards = opts ? std::max(1, opts->n_shards) : 1;
  const int shard = opts ? opts->shard_index : 0;
  if (n_shards > kMaxShards || shard < 0 || shard >= n_shards)
    return fail(PRISM_E_INVALID_ARG, "n_shards must be in [1, 16] and shard_index in [0, n_shards)");
  trace("build: begin");
  Plan plan;
  std::string err;
  prism_status st = PRISM_OK;
  int axis = 0;
  static const int env_rc = [] {
    const char *e = std::getenv("PRISM_REPLICA_CELLS");
    return e ? std::atoi(e) : 1;
  }();
  static const int env_ks = [] {
    const char *e = std::getenv("PRISM_EP_CTA_KS");
    return e ? std::atoi(e) : 0;
  }();
  std::vector<unsigned char> pkey;
  const bool keyed = plan_key(*topo, *tmpl, n_shards, shard, opts ? opts->flags : 0, env_rc, env_ks, pkey);
  const bool cached = keyed && plan_cache_get(pkey, plan, axis);
  if (cached) trace("build: plan from the cache");
  if (!cached) {
    st = plan_graph(*topo, *tmpl, plan, err);
    if (st != PRISM_OK) return fail(st, err);
    trace("build: planned");
    if (n_shards > 1) {
      st = choose_shard_axis(plan, n_shards, opts ? opts->flags : 0, axis, err);
      if (st != PRISM_OK) return fail(st, err);
    }
    {  // replica cells for tp = 1: R = 8 DP replicas per cell when the topology and
       // the shard blocks allow it (PRISM_REPLICA_CELLS=0 keeps one rank per cell: experiments)
      // EP CTAs: the 8 cells of an EP group (R = ep / 8 replicas each) share one CTA, so an EP
      // all-to-all is a register + shared-memory max behind one barrier; a DP-block shard must then
      // hold whole EP groups. PRISM_REPLICA_CELLS=2: replica cells of 8 without EP CTAs.
      const Topo &tt = plan.topo;
      // sixteen cells of ep / 16 replicas when that width is instantiated (2 or 4), else eight
      const int ks = env_ks ? env_ks : ((tt.ep % 16 == 0 && (tt.ep / 16 == 2 || tt.ep / 16 == 4)) ? 16 : 8);
      const bool cta = env_rc != 2 && tt.tp == 1 && tt.ep >= 2 * ks && tt.ep % ks == 0 && tt.ep / ks <= 8 &&
                       (n_shards == 1 || axis == 1 || (tt.dp / n_shards) % tt.ep == 0) &&
                       (ks == 8 || tt.ep / ks == 2 || tt.ep / ks == 4);
      const int R = cta ? tt.ep / ks : 8;
      const bool blocks_ok = n_shards == 1 || axis == 1 || (tt.dp / n_shards) % R == 0;
      // without EP CTAs, plain replica cells when one-rank cells could not all be co-resident (more
      // than ~4k ranks per shard at 28 warps per SM): 8-replica warps instead of the level-by-level
      // fallback
      const int64_t my_ranks = (int64_t)tt.tp * tt.pp * tt.dp / std::max(1, n_shards);
      const bool wide = tt.tp == 1 && my_ranks > 4096;
      if (env_rc && (cta || wide || env_rc == 2) && blocks_ok && replica_cells_ok(tt, R) &&
          (R == 2 || R == 4 || R == 8)) {
        st = plan_replica_cells(plan, R, cta ? ks : 1, err);
        if (st != PRISM_OK) return fail(st, err);
      }
    }
    if (keyed) plan_cache_put(std::move(pkey), plan, axis);
  }

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(PRISM_E_CUDA, "no CUDA device (there is no CPU fallback)");
  auto *G = new prism_graph_s();
  std::unique_ptr<prism_graph_s> guard(G);
  G->device = -1;
  if (opts && opts->device >= 0) CU(cudaSetDevice(opts->device));
  CU(cudaGetDevice(&G->device));
  G->stream = opts ? (cudaStream_t)opts->stream : nullptr;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    G->alloc = g_alloc;
    G->free_fn = g_free;
    G->ctx = g_alloc_ctx;
  }
  G->plan = std::move(plan);
  const Plan &P = G->plan;
  G->tmpl_labels.resize(tmpl->n_ops);
  for (int64_t i = 0; i < tmpl->n_ops; ++i) G->tmpl_labels[i] = tmpl->ops[i].label;
  DevGraph &d = G->dg;
  d.W = (int32_t)P.W;
  d.pp = P.topo.pp;
  d.tp = P.topo.tp;
  d.dp = P.topo.dp;
  d.ep = P.topo.ep;
  d.order = P.topo.order;
  d.N = P.N;
  d.G = P.G;
  d.M = P.M;
  d.nq = (int32_t)P.q.size();
  d.n_shards = n_shards;
  d.shard = shard;
  d.shard_axis = axis;
  d.d0 = axis == 0 ? P.topo.dp / n_shards * shard : 0;
  d.d1 = axis == 0 ? P.topo.dp / n_shards * (shard + 1) : P.topo.dp;
  d.s0 = axis == 1 ? P.topo.pp / n_shards * shard : 0;
  d.s1 = axis == 1 ? P.topo.pp / n_shards * (shard + 1) : P.topo.pp;
  G->n_shards = n_shards;
  G->shard = shard;
  {  // fin rows kept by this graph: a DP block is one contiguous node range under TP_PP_DP (a PP
     // block is not: PP-sharded graphs keep all rows)
    int64_t per_replica = 0;
    for (int s2 = 0; s2 < P.topo.pp; ++s2) per_replica += P.stage_len[s2] * P.topo.tp;
    if (n_shards > 1 && axis == 0 && P.topo.order == PRISM_ORDER_TP_PP_DP) {
      G->fin_node0 = per_replica * d.d0;
      G->fin_rows = per_replica * (d.d1 - d.d0);
    } else {
      G->fin_node0 = 0;
      G->fin_rows = P.N;
    }
    d.fin_node0 = G->fin_node0;
    d.fin_rows = G->fin_rows;
  }
  const size_t W = P.W, N = P.N, M = P.M, Gn = P.G, pp = P.topo.pp;
  const size_t nops = (size_t)tmpl->n_ops;
  // One device allocation for the whole graph (a Python allocator hook costs ~tens of us per
  // call), carved into 256-byte aligned arrays; the host-made tables live in one section that is
  // uploaded with a single copy from a packed host buffer.
  const size_t nslot = P.slot_q.size(), nch = P.chunk_q.size();
  size_t off = 0;
  auto carve = [&off](size_t bytes) {
    off = (off + 255) & ~(size_t)255;
    const size_t o = off;
    off += std::max<size_t>(bytes, 1);
    return o;
  };
  // tables (uploaded)
  const size_t o_tps = carve(nops * 4), o_tsp = carve(nops * 4);
  const size_t o_op0 = carve(pp * 8), o_len = carve(pp * 8), o_slt = carve(pp * 8), o_stat = carve(pp * 8);
  const size_t o_q = carve(P.q.size() * sizeof(QGroup)), o_wpos = carve(P.wpos.size() * 4);
  const size_t o_ss0 = carve(P.stage_slot0.size() * 8), o_slq = carve(nslot * 4), o_sltd = carve(nslot * 4);
  const size_t o_slr = carve(nslot), o_slf = carve(nslot), o_chq = carve(nch * 4), o_chm = carve(nch * 8);
  const size_t o_tcls = carve(nops), o_xptr = carve((pp + 1) * 4), o_xops = carve(P.x_ops.size() * sizeof(XOp));
  const bool ms = P.multistream;
  const size_t o_tq0 = carve(nops * 4);
  // the template fields the expansion copies, as structure-of-arrays (coalesced loads; the 48-byte
  // prism_op records would cost the expander 12 cache lines per warp per field)
  const size_t o_tdur = carve(nops * 8), o_tal = carve(nops * 8), o_tfr = carve(nops * 8), o_tsd = carve(nops * 8);
  const size_t o_tlab = carve(nops * 4), o_tkind = carve(nops), o_tqi = carve(nops * 8);
  const size_t o_tms = ms ? carve(nops * 2) : 0, o_tsp2 = ms ? carve(nops * 4) : 0, o_tes = ms ? carve(nops * 4) : 0;
  const size_t o_crp = P.cell_R > 1 ? carve((pp + 1) * 8) : 0;  // replica cells: cell-record offsets
  const size_t table_bytes = off;
  // graph arrays (written by the expand kernels)
  const size_t o_rp = carve((W + 1) * 4), o_rs = carve((W + 1) * 4), o_rst = carve(W * 4);
  // per node only the structure (rank, previous sync node, slot pointer); a node's duration, kind,
  // label, memory deltas and replay record are its template op's (graph.h nd_*, the cell kernel's
  // record loads), looked up instead of written N times
  const size_t o_nrank = carve(N * 4), o_nps = carve(N * 4), o_ngp = carve((N + 1) * 4);
  const size_t o_ngrp = carve(M * 4), o_gptr = carve((Gn + 1) * 4), o_gmem = carve(M * 4), o_gdur = carve(Gn * 8);
  const size_t o_guid = carve(Gn * 8), o_glvl = carve(Gn * 4), o_nms = carve(M * 4);
  const size_t o_gxb = carve(Gn * 8), o_gli = carve(Gn * 4);
  const size_t o_hb = carve(M * 4), o_hm = carve(M * 4), o_hd = carve(M * 8), o_hu = carve(M * 8);
  const size_t o_hs = n_shards > 1 ? carve(M * 4) : 0;
  const size_t o_nmsk = ms ? carve(N * 2) : 0, o_nsp = ms ? carve(N * 4) : 0, o_nes = ms ? carve(N * 4) : 0;
  const size_t o_words = carve(16);
  const size_t ncrec = P.cell_R > 1 ? (size_t)P.crec_ptr[pp] : 0;
  const size_t o_cb = P.cell_R > 1 ? carve(ncrec * 4) : 0, o_cm = P.cell_R > 1 ? carve(ncrec * 4) : 0;
  const size_t total = off;
  trace("build: tables sized");
  unsigned char *base = G->take<unsigned char>(total);
  trace("build: allocated");
  if (G->oom || !base) return fail(PRISM_E_OOM, "device allocation failed while building the graph");
  auto at = [base](size_t o) { return (void *)(base + o); };
  d.t_prev_sync = (int32_t *)at(o_tps);
  d.t_slot_ptr = (int32_t *)at(o_tsp);
  d.t_op0 = (int64_t *)at(o_op0);
  d.t_len = (int64_t *)at(o_len);
  d.t_slots_total = (int64_t *)at(o_slt);
  d.static_mem = (int64_t *)at(o_stat);
  d.q = (const QGroup *)at(o_q);
  d.wpos = (const int32_t *)at(o_wpos);
  d.stage_slot0 = (const int64_t *)at(o_ss0);
  d.slot_q = (const int32_t *)at(o_slq);
  d.slot_tidx = (const int32_t *)at(o_sltd);
  d.slot_role = (const uint8_t *)at(o_slr);
  d.slot_first = (const uint8_t *)at(o_slf);
  d.chunk_q = (const int32_t *)at(o_chq);
  d.chunk_m = (const int64_t *)at(o_chm);
  d.nchunk = (int32_t)nch;
  d.t_cls = (const uint8_t *)at(o_tcls);
  d.x_ptr = (const int32_t *)at(o_xptr);
  d.x_ops = (const XOp *)at(o_xops);
  d.t_q0 = (const int32_t *)at(o_tq0);
  d.t_dur = (const int64_t *)at(o_tdur);
  d.t_alloc = (const int64_t *)at(o_tal);
  d.t_free = (const int64_t *)at(o_tfr);
  d.t_sdur = (const int64_t *)at(o_tsd);
  d.t_label = (const uint32_t *)at(o_tlab);
  d.t_kind = (const uint8_t *)at(o_tkind);
  d.t_qinfo = (const uint64_t *)at(o_tqi);
  d.ms = ms ? 1 : 0;
  d.ms_streams = P.ms_streams;
  d.ms_events = P.ms_events;
  d.t_ms = ms ? (const uint16_t *)at(o_tms) : nullptr;
  d.t_spred = ms ? (const int32_t *)at(o_tsp2) : nullptr;
  d.t_esrc = ms ? (const int32_t *)at(o_tes) : nullptr;
  d.rank_ptr = (int32_t *)at(o_rp);
  d.rank_slot = (int32_t *)at(o_rs);
  d.rank_stage = (int32_t *)at(o_rst);
  d.node_rank = (int32_t *)at(o_nrank);
  d.node_dur = nullptr;  // template lookups (overrides replace them in dov)
  d.node_kind = nullptr;
  d.node_label = nullptr;
  d.node_alloc = nullptr;
  d.node_free = nullptr;
  d.node_prev_sync = (int32_t *)at(o_nps);
  d.node_gptr = (int32_t *)at(o_ngp);
  d.node_grp = (int32_t *)at(o_ngrp);
  d.grp_ptr = (int32_t *)at(o_gptr);
  d.grp_mem = (int32_t *)at(o_gmem);
  d.grp_dur = (int64_t *)at(o_gdur);
  d.grp_uid = (uint64_t *)at(o_guid);
  d.grp_level = (int32_t *)at(o_glvl);
  d.node_mslot = (int32_t *)at(o_nms);
  d.node_cls = nullptr;
  d.node_sdur = nullptr;
  d.node_uid = nullptr;
  d.grp_xbase = (int64_t *)at(o_gxb);
  d.grp_lidx = (int32_t *)at(o_gli);
  d.h_base = (int32_t *)at(o_hb);
  d.h_meta = (uint32_t *)at(o_hm);
  d.h_dur = (int64_t *)at(o_hd);
  d.h_uid = (uint64_t *)at(o_hu);
  d.h_smask = n_shards > 1 ? (uint32_t *)at(o_hs) : nullptr;
  d.node_ms = ms ? (uint16_t *)at(o_nmsk) : nullptr;
  d.node_spred = ms ? (int32_t *)at(o_nsp) : nullptr;
  d.node_esrc = ms ? (int32_t *)at(o_nes) : nullptr;
  d.M_cross = P.M_cross;
  d.G_large = P.G_large;
  d.cell_R = P.cell_R;
  d.cta_ks = P.cta_ks;
  d.Ltot = (int64_t)nops;
  d.crec_ptr = P.cell_R > 1 ? (const int64_t *)at(o_crp) : nullptr;
  d.c_base = P.cell_R > 1 ? (int32_t *)at(o_cb) : nullptr;
  d.c_meta = P.cell_R > 1 ? (uint32_t *)at(o_cm) : nullptr;
  d.stall_unit = -1;
  d.watchdog_ns = 10ull * 1000 * 1000 * 1000;
  G->words = (uint32_t *)at(o_words);
  cudaStream_t s = G->stream;
  {  // packed upload of the host tables, from a pinned staging buffer when one is available
    PinnedStage ps(table_bytes);
    unsigned char *hb = ps.ptr;
    if (!hb) {  // no pinned memory: pageable fallback (the copy then waits for the stream)
      G->staging.assign(table_bytes, 0);
      hb = G->staging.data();
    }
    // every table below is written in full; the alignment gaps between them are never read
    auto put = [hb](size_t o, const void *src, size_t bytes) {
      if (bytes) std::memcpy(hb + o, src, bytes);
    };
    put(o_tps, P.t_prev_sync.data(), nops * 4);
    put(o_tsp, P.t_slot_ptr.data(), nops * 4);
    put(o_op0, P.stage_op0.data(), pp * 8);
    put(o_len, P.stage_len.data(), pp * 8);
    put(o_slt, P.stage_slots.data(), pp * 8);
    put(o_stat, tmpl->static_mem, pp * 8);
    put(o_q, P.q.data(), P.q.size() * sizeof(QGroup));
    put(o_wpos, P.wpos.data(), P.wpos.size() * 4);
    put(o_ss0, P.stage_slot0.data(), P.stage_slot0.size() * 8);
    put(o_slq, P.slot_q.data(), nslot * 4);
    put(o_sltd, P.slot_tidx.data(), nslot * 4);
    put(o_slr, P.slot_role.data(), nslot);
    put(o_slf, P.slot_first.data(), nslot);
    put(o_chq, P.chunk_q.data(), nch * 4);
    put(o_chm, P.chunk_m.data(), nch * 8);
    put(o_tcls, P.t_cls.data(), nops);
    put(o_tq0, P.t_q0.data(), nops * 4);
    trace("pack: plan tables copied");
    {
      int64_t *tdur = (int64_t *)(hb + o_tdur), *tal = (int64_t *)(hb + o_tal);
      int64_t *tfr = (int64_t *)(hb + o_tfr), *tsd = (int64_t *)(hb + o_tsd);
      uint32_t *tlab = (uint32_t *)(hb + o_tlab);
      uint8_t *tkind = hb + o_tkind;
      uint64_t *tqi = (uint64_t *)(hb + o_tqi);
      for (size_t i = 0; i < nops; ++i) {
        const prism_op &o = tmpl->ops[i];
        tdur[i] = o.dur_ns;
        tal[i] = o.mem_alloc;
        tfr[i] = o.mem_free;
        tlab[i] = o.label;
        tkind[i] = o.kind;
        // replay record duration: a compute span's own, a sync node's first group's (Z2)
        tsd[i] = P.t_q0[i] < 0 ? o.dur_ns : P.q[P.t_q0[i]].dur;
        tqi[i] = 0;
        if (P.t_q0[i] >= 0) {
          const QGroup &q = P.q[P.t_q0[i]];
          tqi[i] = (uint64_t)(q.type & 0xFF) | ((uint64_t)(q.dir & 0xFF) << 8) |
                   ((uint64_t)(q.stage & 0xFFFF) << 16) | ((uint64_t)(uint32_t)q.occ << 32);
        }
      }
    }
    trace("pack: op fields");
    put(o_xptr, P.x_ptr.data(), (pp + 1) * 4);
    if (P.cell_R > 1) put(o_crp, P.crec_ptr.data(), (pp + 1) * 8);
    put(o_xops, P.x_ops.data(), P.x_ops.size() * sizeof(XOp));
    if (ms) {
      put(o_tms, P.t_ms.data(), nops * 2);
      put(o_tsp2, P.t_spred.data(), nops * 4);
      put(o_tes, P.t_esrc.data(), nops * 4);
    }
    trace("build: packed");
    CU(cudaMemcpyAsync(base, hb, table_bytes, cudaMemcpyHostToDevice, s));
    ps.release(s);
    trace("build: upload queued");
  }
  if (opts && (opts->flags & PRISM_BUILD_PROFILE)) {
    G->profile = true;
    for (auto &e : G->ev) CU(cudaEventCreate(&e));
  }
  {  // once per device and process: load every kernel a replay may launch (see replay.cu)
    static std::mutex mu;
    static std::vector<int> loaded;
    std::lock_guard<std::mutex> lk(mu);
    if (std::find(loaded.begin(), loaded.end(), G->device) == loaded.end()) {
      CU(preload_replay_kernels());
      CU(preload_cells());
      CU(preload_rank_kernels());
      CU(preload_peak_kernel());
      loaded.push_back(G->device);
    }
  }
  CU(cudaMemsetAsync(G->words, 0, 16, s));
  if (!(G->h_status = pin_take())) return fail(PRISM_E_OOM, "pinned status words unavailable");
  G->rec(0);
  CU(launch_expand(d, s));
  CU(launch_cell_records(d, s));
  G->rec(1);
  trace("build: expand launched");
  if (!(opts && (opts->flags & PRISM_BUILD_ASYNC))) CU(cudaStreamSynchronize(s));
  *out = guard.release();
  return PRISM_OK;
}

}  // extern "C"

namespace {

// Replay state of one replay (bytes per array; 0 = not needed), carved from the graph's state block.
struct StateReq {
  size_t fin, gfin, rank_end, rslot, acc, rres, sync, part;
};
prism_status ensure_state(prism_graph_t G, const StateReq &q) {
  const size_t want[8] = {q.fin, q.gfin, q.rank_end, q.rslot, q.acc, q.rres, q.sync, q.part};
  size_t off = 0, o[8];
  for (int i = 0; i < 8; ++i) {
    off = (off + 255) & ~(size_t)255;
    o[i] = off;
    off += want[i];
  }
  const size_t total = std::max<size_t>(off, 256);
  bool relayout = false;
  for (int i = 0; i < 8; ++i) relayout |= G->state_off[i] != o[i] || G->state_len[i] != want[i];
  if (total > G->state_cap || !G->state) {
    G->dfree(G->state);
    G->state = (unsigned char *)G->dalloc(total);
    G->state_cap = G->state ? total : 0;
    if (!G->state) return fail(PRISM_E_OOM, "replay-state allocation failed");
    relayout = true;
  }
  // the ready / result slots must be reset when their memory or offsets changed
  if (relayout) G->rslot_dirty = true;
  for (int i = 0; i < 8; ++i) {
    G->state_off[i] = o[i];
    G->state_len[i] = want[i];
  }
  auto at = [&](int i) { return want[i] ? (void *)(G->state + o[i]) : nullptr; };
  G->fin = (int64_t *)at(0);
  G->fin_bytes = want[0];
  G->gfin = (int64_t *)at(1);
  G->gfin_bytes = want[1];
  G->rank_end = (int64_t *)at(2);
  G->rank_end_bytes = want[2];
  G->rslot = (int64_t *)at(3);
  G->rslot_bytes = want[3];
  G->acc = (int64_t *)at(4);
  G->acc_bytes = want[4];
  G->rres = (int64_t *)at(5);
  G->rres_bytes = want[5];
  G->sync_words = (uint32_t *)at(6);
  G->sync_bytes = want[6];
  G->part = (int64_t *)at(7);
  G->part_bytes = want[7];
  return PRISM_OK;
}

// Tiles of every level for a team width of `lanes` (one membership per team per round).
prism_status plan_tiles(prism_graph_s *G, int lanes) {
  if (G->tiles_lanes == lanes) return PRISM_OK;
  const Plan &P = G->plan;
  const int teams = 256 / lanes;
  const int sc = lanes == 32 ? 64 : lanes;
  const int cap_smem = std::max(1, (48 * 1024) / (sc * 8));
  std::vector<Tile> tiles;
  G->lvl_tile_ptr.assign(P.levels + 2, 0);
  G->lvl_max_cnt.assign(P.levels + 2, 1);
  for (int l = 0; l <= P.levels; ++l) {
    G->lvl_tile_ptr[l] = (int32_t)tiles.size();
    for (int32_t qi = P.level_q_ptr[l]; qi < P.level_q_ptr[l + 1]; ++qi) {
      const QGroup &q = P.q[qi];
      int gpt = std::max(1, teams / q.size);
      gpt = std::min(gpt, cap_smem);
      for (int32_t i0 = 0; i0 < q.inst; i0 += gpt) {
        Tile t{qi, i0, std::min(gpt, q.inst - i0), 0};
        G->lvl_max_cnt[l] = std::max(G->lvl_max_cnt[l], t.cnt);
        tiles.push_back(t);
      }
    }
  }
  G->lvl_tile_ptr[P.levels + 1] = (int32_t)tiles.size();
  size_t cap = G->tiles_bytes;
  if (!G->ensure(G->tiles, cap, std::max<size_t>(16, tiles.size() * sizeof(Tile))))
    return fail(PRISM_E_OOM, "tile plan allocation failed");
  G->tiles_bytes = cap;
  if (!tiles.empty()) {
    cudaError_t e = cudaMemcpyAsync(G->tiles, tiles.data(), tiles.size() * sizeof(Tile),
                                    cudaMemcpyHostToDevice, G->stream);
    if (e != cudaSuccess) return fail(PRISM_E_CUDA, cudaGetErrorString(e));
    e = cudaStreamSynchronize(G->stream);  // host vector goes out of scope
    if (e != cudaSuccess) return fail(PRISM_E_CUDA, cudaGetErrorString(e));
  }
  G->tiles_lanes = lanes;
  return PRISM_OK;
}

// One scenario, lane = rank (replay_ranks.cu): scenario stride 1.
prism_status replay_ranks_impl(prism_graph_t G, const prism_scenarios *sc, int64_t *iter_dev) {
  const Plan &P = G->plan;
  ScenParams p{};
  p.S = 1;
  p.first = sc->first;
  p.amp = sc->amp_q16;
  p.seed = sc->seed;
  p.mask = sc->kind_mask;
  p.record = sc->record ? 1 : 0;
  p.mod = 2 * sc->amp_q16 + 1;
  p.mod_magic = ~0ULL / (uint64_t)p.mod + 1;
  p.mod_m32 = p.mod > 1 ? (uint32_t)((((uint64_t)1 << 32) + (uint64_t)p.mod - 1) / (uint64_t)p.mod) : 0xFFFFFFFFu;
  G->recorded = 0;
  const int32_t Sp = 1;
  const size_t lg = std::max<size_t>(16, (size_t)P.G_large * 8);
  const size_t nwords = std::max<size_t>(1, (size_t)P.G_large);
  {
    const StateReq q{p.record ? (size_t)std::max<int64_t>(1, G->fin_rows) * 8 : 0, (size_t)std::max<int64_t>(1, P.G) * 8,
                     (size_t)P.W * 8, std::max<size_t>(16, (size_t)P.M_cross * 8), lg, lg, nwords * 4,
                     segs_scratch_bytes(G->cur(), (int64_t)P.x_ops.size())};
    prism_status st = ensure_state(G, q);
    if (st) return st;
  }
  if (G->rslot_Sp != Sp) G->rslot_dirty = true;
  G->rslot_Sp = Sp;
  if (G->rslot_dirty) {
    CU(cudaMemsetAsync(G->rslot, 0xFF, G->rslot_bytes, G->stream));
    CU(cudaMemsetAsync(G->rres, 0xFF, G->rres_bytes, G->stream));
    G->parity = 0;
    G->rslot_dirty = false;
  }
  CU(launch_replay_guard(G->words, G->rslot, G->rslot_bytes / 8, G->rres, G->rres_bytes / 8, G->parity, G->stream));
  CU(cudaMemsetAsync(G->acc, 0, (size_t)P.G_large * 8, G->stream));
  CU(cudaMemsetAsync(G->sync_words, 0, nwords * 4, G->stream));
  uint32_t *status = G->words;
  G->rec(2);
  int nl = 1;
  CU(launch_ranks(G->cur(), p, G->rslot, G->acc, G->rres, G->sync_words, status, G->parity,
                  p.record ? G->fin : nullptr, G->gfin, G->rank_end, G->part, (int64_t)P.x_ops.size(), &nl,
                  G->stream));
  G->parity ^= 1;
  CU(cudaMemcpyAsync(G->h_status, G->words, 8, cudaMemcpyDeviceToHost, G->stream));
  G->rec(3);
  G->rec(4);
  CU(launch_reduce(P.W, 1, Sp, G->rank_end, iter_dev, G->stream));
  G->rec(5);
  G->launches = 2 + nl;  // guard, rank kernel or segment walk + chain (+ fin walk), reduce
  G->last = p;
  G->last_Sp = Sp;
  G->recorded = p.record;
  G->last_algo = PRISM_ALGO_RANKS;
  return PRISM_OK;
}

prism_status replay_impl(prism_graph_t G, const prism_scenarios *sc, int64_t *iter_dev) {
  if (!G || !sc || !iter_dev) return fail(PRISM_E_INVALID_ARG, "null argument");
  if (sc->n < 1 || sc->n > (1 << 20) || sc->amp_q16 < 0 || sc->amp_q16 > 65535)
    return fail(PRISM_E_INVALID_ARG, "scenario count must be >= 1 and amp_q16 in [0, 65535]");
  if (sc->algo < PRISM_ALGO_AUTO || sc->algo > PRISM_ALGO_RANKS) return fail(PRISM_E_INVALID_ARG, "unknown algo");
  if (sc->first < 0 || (int64_t)sc->first + sc->n > (1LL << 31) - 1)
    return fail(PRISM_E_INVALID_ARG, "first scenario index out of range");
  CU(cudaSetDevice(G->device));
  const int32_t S = sc->n;
  const Plan &P = G->plan;
  // one scenario: the lane = rank kernel when it applies (auto) or is asked for
  // (EP-CTA graphs stay on the cell kernel: its CTA-local all-to-alls beat the rank kernel's
  // global rendezvous even for one scenario)
  if (sc->algo == PRISM_ALGO_RANKS || (sc->algo == PRISM_ALGO_AUTO && S == 1 && G->dg.cta_ks <= 1)) {
    const bool fit = S == 1 && ranks_fit(G->cur(), nullptr);
    if (fit) return replay_ranks_impl(G, sc, iter_dev);
    if (sc->algo == PRISM_ALGO_RANKS)
      return fail(PRISM_E_INVALID_ARG, "PRISM_ALGO_RANKS needs one scenario, an unsharded single-stream graph, "
                                       "tp a power of two <= 32 and co-resident warps");
  }
  // schedule: the cell kernel (64-scenario chunks, one cooperative launch each) when every cell
  // CTA of a chunk can be co-resident, else one launch per frontier level
  const int cell_sc = cells_chunk_scenarios();
  const int cell_chunks = (S + cell_sc - 1) / cell_sc;
  bool cells = false;
  const bool sharded = G->n_shards > 1;
  if (sharded) {
    if (!G->connected) return fail(PRISM_E_INVALID_ARG, "sharded graph: call prism_shard_prepare and prism_shard_connect first");
    if (G->local_group)
      return fail(PRISM_E_INVALID_ARG, "shards on one device replay together in one cooperative launch "
                                       "(prism_replay_local_shards): separate launches are not guaranteed to run concurrently");
    if (S != G->ex_S) return fail(PRISM_E_INVALID_ARG, "sharded graph: the replay's scenario count must equal prism_shard_prepare's");
    if (sc->algo == PRISM_ALGO_LEVELS) return fail(PRISM_E_INVALID_ARG, "sharded replays run on the cell kernel only");
    if (!cells_fit(G->cur(), cell_chunks)) return fail(PRISM_E_INVALID_ARG, "sharded replay: the shard's cells do not fit co-resident on the device");
  }
  if (sc->algo != PRISM_ALGO_LEVELS) {
    cells = cells_fit(G->cur(), cell_chunks);
    if (!cells && sc->algo == PRISM_ALGO_CELLS)
      return fail(PRISM_E_INVALID_ARG, "PRISM_ALGO_CELLS: the cells of this graph do not fit co-resident on the device");
  }
  if (!cells && G->plan.multistream)
    return fail(PRISM_E_INVALID_ARG, "multi-stream graphs (row f2) replay on the cell kernel only (tp <= 8, "
                                     "cells co-resident)");
  int lanes = 32;
  if (!cells)
    for (lanes = 1; lanes < S && lanes < 32;) lanes <<= 1;
  const int SC = cells ? cell_sc : (lanes == 32 ? 64 : lanes);
  const int nchunks = (S + SC - 1) / SC;
  const int32_t Sp = nchunks * SC;
  ScenParams p{};
  p.S = S;
  p.first = sc->first;
  p.amp = sc->amp_q16;
  p.seed = sc->seed;
  p.mask = sc->kind_mask;
  p.record = sc->record ? 1 : 0;
  p.mod = 2 * sc->amp_q16 + 1;
  p.mod_magic = ~0ULL / (uint64_t)p.mod + 1;
  p.mod_m32 = p.mod > 1 ? (uint32_t)((((uint64_t)1 << 32) + (uint64_t)p.mod - 1) / (uint64_t)p.mod) : 0xFFFFFFFFu;
  G->recorded = 0;
  G->gathered_k = -1;
  trace("replay: begin");
  {
    StateReq q{p.record ? (size_t)std::max<int64_t>(1, G->fin_rows) * Sp * 8 : 0, (size_t)std::max<int64_t>(1, P.G) * Sp * 8,
               (size_t)P.W * Sp * 8, 0, 0, 0, 0, 0};
    if (sharded) {
      q.part = (size_t)Sp * 8;
    } else if (cells) {
      q.rslot = std::max<size_t>(16, (size_t)P.M_cross * Sp * 8);
      q.acc = q.rres = std::max<size_t>(16, (size_t)P.G_large * Sp * 8);
      q.sync = std::max<size_t>(1, (size_t)P.G_large * nchunks) * 4;
    }
    prism_status st = ensure_state(G, q);
    if (st) return st;
  }
  int64_t launches = 0;
  trace("replay: buffers ready");
  if (sharded) {
    // row e: ready slots / accumulators / counters live in the peer-mapped exchange buffer; they
    // were reset at prepare, and the accumulators and counters are reset again right after the
    // cell kernel, before this shard publishes its partial (the peers' next pushes wait for it)
    // an abort leaves the peers' exchange state inconsistent: the graph is re-prepared instead of
    // reset (check_status disconnects it), so the guard only folds the status
    CU(launch_replay_guard(G->words, nullptr, 0, nullptr, 0, G->parity, G->stream));
    ++launches;
    G->link.epoch += 1;
    uint32_t *status = G->words;
    int64_t *rslot = (int64_t *)(G->ex + G->link.o_rslot);
    int64_t *acc = (int64_t *)(G->ex + G->link.o_acc);
    uint32_t *arrive = (uint32_t *)(G->ex + G->link.o_arrive);
    G->rec(2);
    trace("shard: launch cells");
    const int per_launch = cells_chunks_per_launch(G->cur(), nchunks);
    for (int ch = 0; ch < nchunks; ch += per_launch) {
      CU(launch_cells(G->cur(), p, rslot, acc, nullptr, arrive, status, G->parity, p.record ? G->fin : nullptr,
                      G->gfin, G->rank_end, ch, std::min(per_launch, nchunks - ch), Sp, &G->link, G->stream));
      ++launches;
    }
    trace("shard: cells launched");
    G->parity ^= 1;
    CU(cudaMemsetAsync(acc, 0, (size_t)P.G_large * Sp * 8, G->stream));
    CU(cudaMemsetAsync(arrive, 0, (size_t)P.G_large * nchunks * 4, G->stream));
    trace("shard: memsets");
    G->rec(3);
    G->rec(4);
    CU(launch_shard_reduce(G->cur(), G->link, S, Sp, G->rank_end, G->part, iter_dev, status, G->stream));
    trace("shard: reduce launched");
    CU(cudaMemcpyAsync(G->h_status, G->words, 8, cudaMemcpyDeviceToHost, G->stream));
    trace("shard: status copy");
    launches += 2;
  } else if (cells) {
    if (G->rslot_Sp != Sp) G->rslot_dirty = true;
    G->rslot_Sp = Sp;
    const size_t nwords = G->sync_bytes / 4;
    if (G->rslot_dirty) {  // all slots read "not yet" under parity 0
      CU(cudaMemsetAsync(G->rslot, 0xFF, G->rslot_bytes, G->stream));
      CU(cudaMemsetAsync(G->rres, 0xFF, G->rres_bytes, G->stream));
      G->parity = 0;
      G->rslot_dirty = false;
    }
    CU(launch_replay_guard(G->words, G->rslot, G->rslot_bytes / 8, G->rres, G->rres_bytes / 8, G->parity, G->stream));
    ++launches;
    CU(cudaMemsetAsync(G->acc, 0, (size_t)P.G_large * Sp * 8, G->stream));
    CU(cudaMemsetAsync(G->sync_words, 0, nwords * 4, G->stream));
    G->rec(2);
    uint32_t *status = G->words;
    const int per_launch = cells_chunks_per_launch(G->cur(), nchunks);
    for (int ch = 0; ch < nchunks; ch += per_launch) {
      CU(launch_cells(G->cur(), p, G->rslot, G->acc, G->rres, G->sync_words, status, G->parity,
                      p.record ? G->fin : nullptr, G->gfin, G->rank_end, ch,
                      std::min(per_launch, nchunks - ch), Sp, nullptr, G->stream));
      ++launches;
    }
    G->parity ^= 1;
    CU(cudaMemcpyAsync(G->h_status, G->words, 8, cudaMemcpyDeviceToHost, G->stream));
    G->rec(3);
    G->rec(4);
  } else {
    prism_status st = plan_tiles(G, lanes);
    if (st) return st;
    G->rec(2);
    for (int l = 1; l <= P.levels; ++l) {
      const int32_t t0 = G->lvl_tile_ptr[l], t1 = G->lvl_tile_ptr[l + 1];
      if (t1 == t0) continue;
      CU(launch_level(G->cur(), p, G->tiles + t0, t1 - t0, G->lvl_max_cnt[l], p.record ? G->fin : nullptr,
                      G->gfin, lanes, nchunks, G->stream));
      ++launches;
    }
    G->rec(3);
    CU(launch_tail(G->cur(), p, p.record ? G->fin : nullptr, G->gfin, G->rank_end, lanes, nchunks, G->stream));
    G->rec(4);
    ++launches;
  }
  if (!sharded) {
    CU(launch_reduce(G->cur().W, S, Sp, G->rank_end, iter_dev, G->stream));
    ++launches;
  }
  G->rec(5);
  G->launches = launches;
  G->last = p;
  G->last_Sp = Sp;
  G->recorded = p.record;
  G->last_algo = cells ? PRISM_ALGO_CELLS : PRISM_ALGO_LEVELS;
  return PRISM_OK;
}

// Abort status of the waiting replays queued so far (valid once the stream has passed them, i.e.
// after a stream synchronisation): the last one's word and the sticky first abort of the earlier
// ones (folded by the next replay's guard kernel). Reported once, then cleared on both sides.
prism_status check_status(prism_graph_t G) {
  if (!G->h_status) return PRISM_OK;
  const uint32_t s = G->h_status[1] ? G->h_status[1] : G->h_status[0];
  if (s == 0) return PRISM_OK;
  G->h_status[0] = G->h_status[1] = 0;
  G->recorded = 0;
  G->rslot_dirty = true;
  G->connected = false;  // a sharded graph must be re-prepared after an aborted replay
  cudaMemsetAsync(G->words, 0, 8, G->stream);  // stream is idle here (synchronised by the caller)
  cudaStreamSynchronize(G->stream);
  char b[160];
  std::snprintf(b, sizeof b, "replay aborted by the device watchdog (no progress for %.3f s); results of the "
                "replays since the last synchronising call are invalid", (double)G->dg.watchdog_ns * 1e-9);
  return fail((prism_status)s, b);
}

}  // namespace

extern "C" {

prism_status prism_replay_async(prism_graph_t G, const prism_scenarios *sc, int64_t *iter_ns_dev_out) {
  return replay_impl(G, sc, iter_ns_dev_out);
}

prism_status prism_replay(prism_graph_t G, const prism_scenarios *sc, int64_t *iter_ns_out) {
  if (!G || !sc || !iter_ns_out) return fail(PRISM_E_INVALID_ARG, "null argument");
  if (sc->n < 1) return fail(PRISM_E_INVALID_ARG, "scenario count must be >= 1");
  CU(cudaSetDevice(G->device));
  if (!G->ensure(G->iter, G->iter_bytes, (size_t)sc->n * 8)) return fail(PRISM_E_OOM, "iter allocation failed");
  prism_status st = replay_impl(G, sc, G->iter);
  if (st) return st;
  CU(cudaMemcpyAsync(iter_ns_out, G->iter, (size_t)sc->n * 8, cudaMemcpyDeviceToHost, G->stream));
  CU(cudaStreamSynchronize(G->stream));
  return check_status(G);
}

// What a reader of the recorded times (query, critical path, time-ordered peak) sees for scenario
// k: the graph's own fin / gfin, or — for a sharded graph after prism_shard_gather(k) — the gather
// columns (every rank's finishes of that one scenario: the Sp = 1 layout, all rows, local index 0,
// perturbation key shifted to the gathered scenario).
struct ReadView {
  DevGraph g;
  ScenParams p;
  const int64_t *fin, *gfin;
  int32_t Sp, k;
};
static ReadView read_view(prism_graph_t G, int32_t scenario) {
  ReadView v{G->cur(), G->last, G->fin, G->gfin, G->last_Sp, scenario};
  if (G->n_shards > 1 && G->gathered_k == scenario && G->ex) {
    v.g.fin_node0 = 0;
    v.g.fin_rows = G->plan.N;
    v.p.first = G->last.first + scenario;
    v.fin = (const int64_t *)(G->ex + G->link.o_gcol);
    v.gfin = (const int64_t *)(G->ex + G->link.o_ggcol);
    v.Sp = 1;
    v.k = 0;
  }
  return v;
}

// Peak memory into a device array: program order (single-stream graphs, any time) or, for
// multi-stream graphs and prism_peak_memory_at, time order of `scenario` of the recorded replay.
static prism_status peak_impl(prism_graph_t G, int32_t scenario, bool time_ordered, int64_t *peak_dev) {
  const Plan &P = G->plan;
  if (!time_ordered) {
    G->rec(6);
    CU(launch_peak(G->cur(), peak_dev, G->stream));
    G->rec(7);
    return PRISM_OK;
  }
  if (!G->recorded)
    return fail(PRISM_E_NOT_REPLAYED, "time-ordered peak memory needs a replay with record != 0 (multi-stream graphs)");
  if (scenario < 0 || scenario >= G->last.S) return fail(PRISM_E_INVALID_ARG, "scenario outside the last replay");
  if (G->n_shards > 1 && G->gathered_k != scenario)
    return fail(PRISM_E_INVALID_ARG, "sharded graph: gather the scenario first (prism_shard_gather)");
  const ReadView v = read_view(G, scenario);
  int64_t max_len = 0;
  for (int s = 0; s < P.topo.pp; ++s) max_len = std::max(max_len, P.stage_len[s]);
  if (max_len > kMaxTimeOrderedOps)
    return fail(PRISM_E_INVALID_ARG, "time-ordered peak memory supports at most 4096 ops per rank");
  uint32_t *status = G->words + 2;
  CU(cudaMemsetAsync(status, 0, 4, G->stream));
  G->rec(6);
  CU(launch_peak_time(v.g, v.p, v.Sp, v.fin, v.gfin, v.k, (int32_t)max_len,
                      peak_dev, status, G->stream));
  G->rec(7);
  CU(cudaMemcpyAsync(G->h_status + 2, status, 4, cudaMemcpyDeviceToHost, G->stream));
  return PRISM_OK;
}

// Status of the time-ordered memory scans queued so far (after a stream synchronisation).
static prism_status memory_status(prism_graph_t G) {
  if (G->h_status && G->h_status[2] != 0) {
    const uint32_t s = G->h_status[2];
    G->h_status[2] = 0;
    return fail((prism_status)s, "a rank's running allocation drops below zero in time order");
  }
  return PRISM_OK;
}

prism_status prism_sync(prism_graph_t G) {
  if (!G) return fail(PRISM_E_INVALID_ARG, "null graph");
  CU(cudaSetDevice(G->device));
  CU(cudaStreamSynchronize(G->stream));
  prism_status st = check_status(G);
  const prism_status ms = memory_status(G);
  return st ? st : ms;
}

prism_status prism_debug_set(prism_graph_t G, int32_t key, int64_t value) {
  if (!G) return fail(PRISM_E_INVALID_ARG, "null graph");
  switch (key) {
    case PRISM_DEBUG_WATCHDOG_NS:
      if (value < 1000) return fail(PRISM_E_INVALID_ARG, "watchdog must be >= 1 us");
      G->dg.watchdog_ns = G->dov.watchdog_ns = (uint64_t)value;
      return PRISM_OK;
    case PRISM_DEBUG_STALL_UNIT:
      if (value < -1 || value > INT32_MAX) return fail(PRISM_E_INVALID_ARG, "stall unit out of range");
      G->dg.stall_unit = G->dov.stall_unit = (int32_t)value;
      return PRISM_OK;
    default: return fail(PRISM_E_INVALID_ARG, "unknown debug key");
  }
}

prism_status prism_peak_memory_async(prism_graph_t G, int64_t *peak_dev) {
  if (!G || !peak_dev) return fail(PRISM_E_INVALID_ARG, "null argument");
  CU(cudaSetDevice(G->device));
  return peak_impl(G, 0, G->plan.multistream, peak_dev);
}

static prism_status peak_host(prism_graph_t G, int32_t scenario, bool time_ordered, int64_t *peak_out) {
  CU(cudaSetDevice(G->device));
  const size_t bytes = std::max<size_t>(16, (size_t)G->plan.W * 8);
  if (!G->ensure(G->scratch, G->scratch_bytes, bytes)) return fail(PRISM_E_OOM, "scratch allocation failed");
  prism_status st = peak_impl(G, scenario, time_ordered, G->scratch);
  if (st) return st;
  CU(cudaMemcpyAsync(peak_out, G->scratch, (size_t)G->plan.W * 8, cudaMemcpyDeviceToHost, G->stream));
  CU(cudaStreamSynchronize(G->stream));
  return memory_status(G);
}

prism_status prism_peak_memory(prism_graph_t G, int64_t *peak_out) {
  if (!G || !peak_out) return fail(PRISM_E_INVALID_ARG, "null argument");
  return peak_host(G, 0, G->plan.multistream, peak_out);
}

prism_status prism_peak_memory_at(prism_graph_t G, int32_t scenario, int64_t *peak_out) {
  if (!G || !peak_out) return fail(PRISM_E_INVALID_ARG, "null argument");
  return peak_host(G, scenario, true, peak_out);
}

prism_status prism_query_rank(prism_graph_t G, int32_t rank, int32_t scenario, int64_t *start_ns,
                              int64_t *finish_ns, int64_t cap, int64_t *n_ops_out,
                              int32_t coords_out[5]) {
  if (!G) return fail(PRISM_E_INVALID_ARG, "null graph");
  const Plan &P = G->plan;
  if (rank < 0 || rank >= P.W) return fail(PRISM_E_UNKNOWN_RANK, "rank " + std::to_string(rank) + " outside the world");
  const Topo &t = P.topo;
  int32_t tp_i = rank % t.tp, pp_i, dp_i;
  if (t.order == PRISM_ORDER_MEGATRON) {
    dp_i = (rank / t.tp) % t.dp;
    pp_i = rank / (t.tp * t.dp);
  } else {
    pp_i = (rank / t.tp) % t.pp;
    dp_i = rank / (t.tp * t.pp);
  }
  if (coords_out) {
    coords_out[0] = tp_i;
    coords_out[1] = pp_i;
    coords_out[2] = dp_i;
    coords_out[3] = dp_i % t.ep;
    coords_out[4] = dp_i / t.ep;
  }
  const int64_t n = P.stage_len[pp_i];
  if (n_ops_out) *n_ops_out = n;
  if (G->n_shards > 1 && start_ns && G->gathered_k != scenario &&
      (dp_i < G->dg.d0 || dp_i >= G->dg.d1 || pp_i < G->dg.s0 || pp_i >= G->dg.s1))
    return fail(PRISM_E_INVALID_ARG, "rank " + std::to_string(rank) + " is replayed by shard " +
                                         std::to_string(G->dg.shard_axis == 1 ? pp_i / (t.pp / G->n_shards)
                                                                              : dp_i / (t.dp / G->n_shards)));
  if (!G->recorded) return fail(PRISM_E_NOT_REPLAYED, "no replay with record != 0 has run on this graph");
  if (scenario < 0 || scenario >= G->last.S) return fail(PRISM_E_INVALID_ARG, "scenario outside the last replay");
  if (cap < n || (n > 0 && (!start_ns || !finish_ns))) return fail(PRISM_E_INVALID_ARG, "output capacity too small");
  if (n == 0) return PRISM_OK;
  CU(cudaSetDevice(G->device));
  const size_t bytes = (size_t)n * 16;
  if (!G->ensure(G->scratch, G->scratch_bytes, bytes)) return fail(PRISM_E_OOM, "scratch allocation failed");
  const ReadView v = read_view(G, scenario);
  CU(launch_query(v.g, v.p, v.Sp, v.fin, v.gfin, rank, v.k, G->scratch,
                  G->scratch + n, G->stream));
  CU(cudaMemcpyAsync(start_ns, G->scratch, (size_t)n * 8, cudaMemcpyDeviceToHost, G->stream));
  CU(cudaMemcpyAsync(finish_ns, G->scratch + n, (size_t)n * 8, cudaMemcpyDeviceToHost, G->stream));
  CU(cudaStreamSynchronize(G->stream));
  return check_status(G);
}

// ---- rows f1 / f3 / f4: per-node durations and memory deltas, critical path ---------------

}  // extern "C"

namespace {

// Layout helper of the override blocks (256-byte aligned arrays in one allocation).
struct Carve {
  size_t off = 0;
  size_t operator()(size_t bytes) {
    off = (off + 255) & ~(size_t)255;
    const size_t o = off;
    off += std::max<size_t>(bytes, 8);
    return o;
  }
};

// Recomputes the derived per-node arrays from the set_durations inputs `din` and the MoE load `me`
// into a new block; on success it replaces the graph's block (stream-ordered free of the old one,
// which earlier replays may still read), else the graph keeps its previous overrides.
prism_status apply_overrides(prism_graph_t G, const DurIn &din, bool din_any, const MoeIn &me) {
  const Plan &P = G->plan;
  if (!din_any && me.n_events == 0) {
    G->ov_active = false;
    G->recorded = 0;
    return PRISM_OK;
  }
  const int64_t N = P.N, Gn = P.G, M = P.M;
  const bool mem = din.al || din.fr || (me.n_events > 0 && (me.scale & (PRISM_MOE_ALLOC | PRISM_MOE_FREE)));
  Carve c;
  const size_t o_eff = c(N * 8), o_gd = c(Gn * 8), o_sd = c(N * 8), o_hd = c(M * 8);
  const size_t o_al = mem ? c(N * 8) : 0, o_fr = mem ? c(N * 8) : 0;
  unsigned char *B = (unsigned char *)G->dalloc(c.off);
  if (!B) return fail(PRISM_E_OOM, "duration override allocation failed");
  cudaStream_t st = G->stream;
  int64_t *eff = (int64_t *)(B + o_eff), *gdur = (int64_t *)(B + o_gd), *sdur = (int64_t *)(B + o_sd);
  int64_t *hdur = (int64_t *)(B + o_hd);
  int64_t *eal = mem ? (int64_t *)(B + o_al) : nullptr, *efr = mem ? (int64_t *)(B + o_fr) : nullptr;
  uint32_t *status = G->words + 3;
  cudaError_t e = cudaMemsetAsync(status, 0, 4, st);
  if (e == cudaSuccess) e = launch_durations(G->dg, din, me, eff, eal, efr, gdur, sdur, hdur, status, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(G->h_status + 3, status, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    G->dfree(B);
    return fail(PRISM_E_CUDA, std::string("override kernels: ") + cudaGetErrorString(e));
  }
  const uint32_t bad = G->h_status[3];
  if (bad) {
    G->dfree(B);
    return fail((prism_status)bad, bad == PRISM_E_NEGATIVE_MEMORY
                                       ? "a rank's running allocation drops below zero (program order)"
                                       : "a per-node duration / memory delta is out of range (duration [0, 2^40], "
                                         "memory [0, 2^43])");
  }
  G->dfree(G->ov);
  G->ov = B;
  DevGraph &dv = G->dov;
  dv = G->dg;
  dv.node_dur = eff;
  dv.grp_dur = gdur;
  dv.node_sdur = sdur;
  dv.h_dur = hdur;
  if (mem) {
    dv.node_alloc = eal;
    dv.node_free = efr;
  }
  dv.per_rank_dur = 1;
  G->ov_active = true;
  G->recorded = 0;
  return PRISM_OK;
}

}  // namespace

extern "C" {

prism_status prism_set_durations(prism_graph_t G, const prism_durations *d) {
  if (!G) return fail(PRISM_E_INVALID_ARG, "null graph");
  CU(cudaSetDevice(G->device));
  const Plan &P = G->plan;
  const bool any = d && (d->node_dur || d->n_labels > 0 || d->rank_slow_q16 || d->node_alloc || d->node_free);
  if (!any) {
    prism_status st = apply_overrides(G, DurIn{}, false, G->moe);
    if (st) return st;
    G->dfree(G->din_blk);
    G->din_blk = nullptr;
    G->din = DurIn{};
    G->din_any = false;
    return PRISM_OK;
  }
  const int64_t N = P.N, W = P.W;
  if (d->n_labels < 0 || (d->n_labels > 0 && (!d->labels || !d->label_dur)))
    return fail(PRISM_E_INVALID_ARG, "label overrides: n_labels >= 0 with both arrays");
  // host validation of the small inputs (per-node arrays are checked on the device)
  std::vector<std::pair<uint32_t, int64_t>> lab;
  if (d->n_labels > 0) {
    std::vector<uint32_t> have;
    have.reserve(64);
    for (int s = 0; s < P.topo.pp; ++s)  // every template op is instantiated on tp*dp >= 1 ranks
      for (int64_t i = 0; i < P.stage_len[s]; ++i) have.push_back(G->tmpl_labels[P.stage_op0[s] + i]);
    std::sort(have.begin(), have.end());
    for (int32_t i = 0; i < d->n_labels; ++i) {
      if (d->label_dur[i] < 0 || d->label_dur[i] > (1LL << 40)) return fail(PRISM_E_INVALID_ARG, "label duration outside [0, 2^40]");
      if (!std::binary_search(have.begin(), have.end(), d->labels[i])) {
        char b[64];
        std::snprintf(b, sizeof b, "no node carries label 0x%x", d->labels[i]);
        return fail(PRISM_E_UNKNOWN_LABEL, b);
      }
      lab.emplace_back(d->labels[i], d->label_dur[i]);
    }
    std::sort(lab.begin(), lab.end());
    for (size_t i = 1; i < lab.size(); ++i)
      if (lab[i].first == lab[i - 1].first) return fail(PRISM_E_INVALID_ARG, "duplicate label override");
  }
  if (d->rank_slow_q16)
    for (int64_t r = 0; r < W; ++r)
      if (d->rank_slow_q16[r] < 0 || d->rank_slow_q16[r] > (1 << 20))
        return fail(PRISM_E_INVALID_ARG, "rank_slow_q16 outside [0, 2^20] (a factor of at most 16)");
  const size_t L = lab.size();
  Carve c;
  const size_t o_base = d->node_dur ? c(N * 8) : 0, o_lab = c(L * 4), o_ldur = c(L * 8);
  const size_t o_rf = d->rank_slow_q16 ? c(W * 4) : 0;
  const size_t o_al = d->node_alloc ? c(N * 8) : 0, o_fr = d->node_free ? c(N * 8) : 0;
  unsigned char *B = (unsigned char *)G->dalloc(c.off);
  if (!B) return fail(PRISM_E_OOM, "duration override allocation failed");
  cudaStream_t st = G->stream;
  std::vector<uint32_t> hl(L);
  std::vector<int64_t> hd(L);
  for (size_t i = 0; i < L; ++i) {
    hl[i] = lab[i].first;
    hd[i] = lab[i].second;
  }
  cudaError_t e = cudaSuccess;
  // cudaMemcpyDefault (unified addressing): node_dur / node_alloc / node_free may be device arrays
  // (measured durations already on the GPU: a device-to-device copy instead of a pageable upload)
  auto up = [&](size_t o, const void *src, size_t bytes) {
    if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(B + o, src, bytes, cudaMemcpyDefault, st);
  };
  if (d->node_dur) up(o_base, d->node_dur, N * 8);
  up(o_lab, hl.data(), L * 4);
  up(o_ldur, hd.data(), L * 8);
  if (d->rank_slow_q16) up(o_rf, d->rank_slow_q16, W * 4);
  if (d->node_alloc) up(o_al, d->node_alloc, N * 8);
  if (d->node_free) up(o_fr, d->node_free, N * 8);
  if (e != cudaSuccess) {
    G->dfree(B);
    return fail(PRISM_E_CUDA, cudaGetErrorString(e));
  }
  DurIn in{};
  in.base = d->node_dur ? (const int64_t *)(B + o_base) : nullptr;
  in.labels = (const uint32_t *)(B + o_lab);
  in.label_dur = (const int64_t *)(B + o_ldur);
  in.n_labels = (int32_t)L;
  in.rank_f = d->rank_slow_q16 ? (const int32_t *)(B + o_rf) : nullptr;
  in.al = d->node_alloc ? (const int64_t *)(B + o_al) : nullptr;
  in.fr = d->node_free ? (const int64_t *)(B + o_fr) : nullptr;
  prism_status s2 = apply_overrides(G, in, true, G->moe);  // synchronizes: the host arrays may go away
  if (s2) {
    G->dfree(B);
    return s2;
  }
  G->dfree(G->din_blk);
  G->din_blk = B;
  G->din = in;
  G->din_any = true;
  return PRISM_OK;
}

prism_status prism_set_moe_load(prism_graph_t G, const prism_moe_load *m) {
  if (!G) return fail(PRISM_E_INVALID_ARG, "null graph");
  CU(cudaSetDevice(G->device));
  const Plan &P = G->plan;
  if (!m || m->n_events == 0) {
    prism_status st = apply_overrides(G, G->din, G->din_any, MoeIn{});
    if (st) return st;
    G->dfree(G->moe_blk);
    G->moe_blk = nullptr;
    G->moe = MoeIn{};
    return PRISM_OK;
  }
  if (m->n_events < 0 || !m->op_event || !m->br_q16) return fail(PRISM_E_INVALID_ARG, "MoE load: n_events >= 0 with both arrays");
  if (m->scale & ~(uint32_t)(PRISM_MOE_DUR | PRISM_MOE_ALLOC | PRISM_MOE_FREE))
    return fail(PRISM_E_INVALID_ARG, "MoE load: unknown scale bits");
  const int64_t nops = (int64_t)G->tmpl_labels.size(), ep = P.topo.ep;
  for (int64_t i = 0; i < nops; ++i)
    if (m->op_event[i] < -1 || m->op_event[i] >= m->n_events)
      return fail(PRISM_E_INVALID_ARG, "op_event[" + std::to_string(i) + "] outside [-1, n_events)");
  const int64_t nbr = (int64_t)m->n_events * ep;
  for (int64_t i = 0; i < nbr; ++i)
    if (m->br_q16[i] < 0 || m->br_q16[i] > (1 << 20))
      return fail(PRISM_E_INVALID_ARG, "br_q16[" + std::to_string(i) + "] outside [0, 2^20]");
  Carve c;
  const size_t o_ev = c(nops * 4), o_br = c(nbr * 4);
  unsigned char *B = (unsigned char *)G->dalloc(c.off);
  if (!B) return fail(PRISM_E_OOM, "MoE load allocation failed");
  cudaError_t e = cudaMemcpyAsync(B + o_ev, m->op_event, nops * 4, cudaMemcpyHostToDevice, G->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(B + o_br, m->br_q16, nbr * 4, cudaMemcpyHostToDevice, G->stream);
  if (e != cudaSuccess) {
    G->dfree(B);
    return fail(PRISM_E_CUDA, cudaGetErrorString(e));
  }
  MoeIn me{(const int32_t *)(B + o_ev), (const int32_t *)(B + o_br), m->n_events, m->scale};
  prism_status st = apply_overrides(G, G->din, G->din_any, me);
  if (st) {
    G->dfree(B);
    return st;
  }
  G->dfree(G->moe_blk);
  G->moe_blk = B;
  G->moe = me;
  return PRISM_OK;
}

prism_status prism_critical_path(prism_graph_t G, int32_t scenario, int32_t *path_out, int64_t cap,
                                 int64_t *n_out, int64_t *T_out) {
  if (!G || !n_out) return fail(PRISM_E_INVALID_ARG, "null argument");
  if (!G->recorded) return fail(PRISM_E_NOT_REPLAYED, "no replay with record != 0 has run on this graph");
  if (scenario < 0 || scenario >= G->last.S) return fail(PRISM_E_INVALID_ARG, "scenario outside the last replay");
  if (G->n_shards > 1 && G->gathered_k != scenario)
    return fail(PRISM_E_INVALID_ARG, "sharded graph: gather the scenario first (prism_shard_gather)");
  if (cap < 0 || (cap > 0 && !path_out)) return fail(PRISM_E_INVALID_ARG, "bad path capacity");
  CU(cudaSetDevice(G->device));
  const Plan &P = G->plan;
  const int64_t pc = std::min<int64_t>(cap, P.N + 1);
  const ReadView v = read_view(G, scenario);
  // [S iter][the kernels' scratch (crit_scratch_bytes)]
  const size_t need = (size_t)G->last.S * 8 + 64 + crit_scratch_bytes(v.g, pc);
  if (!G->ensure(G->crit, G->crit_bytes, need)) return fail(PRISM_E_OOM, "critical-path scratch allocation failed");
  int64_t *iter = (int64_t *)G->crit;
  void *scratch = (void *)(((uintptr_t)(iter + G->last.S) + 63) & ~(uintptr_t)63);
  // T: the unsharded replay's rank ends (multi-stream ranks included) reduce to it directly
  const bool have_T = G->n_shards == 1;
  if (have_T) CU(launch_reduce(P.W, G->last.S, G->last_Sp, G->rank_end, iter, G->stream));
  int32_t *pls[3];
  CU(launch_critical_path(v.g, v.p, v.fin, v.Sp, v.k, iter, have_T, scratch, pls, pc, G->stream));
  int32_t *path = pls[0];
  int64_t *len = (int64_t *)pls[1];
  int64_t hl = 0, hT = 0;
  CU(cudaMemcpyAsync(&hl, len, 8, cudaMemcpyDeviceToHost, G->stream));
  CU(cudaMemcpyAsync(&hT, iter + v.k, 8, cudaMemcpyDeviceToHost, G->stream));
  CU(cudaStreamSynchronize(G->stream));
  *n_out = hl;
  if (T_out) *T_out = hT;
  if (hl > cap) return fail(PRISM_E_INVALID_ARG, "path capacity too small: need " + std::to_string(hl));
  if (hl > 0) {
    CU(cudaMemcpyAsync(path_out, path, (size_t)hl * 4, cudaMemcpyDeviceToHost, G->stream));
    CU(cudaStreamSynchronize(G->stream));
  }
  return check_status(G);
}

// ---- row e: sharding ---------------------------------------------------------------------

prism_status prism_replay_local_shards(const prism_graph_t *shards, int32_t n, const prism_scenarios *sc,
                                       int64_t *iter_dev) {
  if (!shards || !sc || !iter_dev || n < 2 || n > kMaxShards) return fail(PRISM_E_INVALID_ARG, "bad arguments");
  prism_graph_t G0 = shards[0];
  for (int i = 0; i < n; ++i) {
    const prism_graph_t G = shards[i];
    if (!G || G->n_shards != n || G->shard != i || !G->connected || !G->local_group || G->device != G0->device ||
        G->ex_S != sc->n || G->parity != G0->parity || G->plan.W != G0->plan.W || G->ov_active != G0->ov_active)
      return fail(PRISM_E_INVALID_ARG, "shard " + std::to_string(i) + " is not a connected local shard of this group "
                                       "(same device, prepared for this scenario count, replayed together)");
  }
  if (sc->amp_q16 < 0 || sc->amp_q16 > 65535 || sc->algo == PRISM_ALGO_LEVELS || sc->algo == PRISM_ALGO_RANKS ||
      sc->first < 0 || (int64_t)sc->first + sc->n > (1LL << 31) - 1)
    return fail(PRISM_E_INVALID_ARG, "bad scenario batch for a sharded replay (cell kernel only)");
  CU(cudaSetDevice(G0->device));
  const Plan &P = G0->plan;
  const int32_t S = sc->n;
  const int SC = cells_chunk_scenarios();
  const int nchunks = (S + SC - 1) / SC;
  const int32_t Sp = nchunks * SC;
  if (!cells_fit(G0->cur(), nchunks, n))
    return fail(PRISM_E_INVALID_ARG, "the local shards' cells do not fit co-resident on the device");
  ScenParams p{};
  p.S = S;
  p.first = sc->first;
  p.amp = sc->amp_q16;
  p.seed = sc->seed;
  p.mask = sc->kind_mask;
  p.record = sc->record ? 1 : 0;
  p.mod = 2 * sc->amp_q16 + 1;
  p.mod_magic = ~0ULL / (uint64_t)p.mod + 1;
  p.mod_m32 = p.mod > 1 ? (uint32_t)((((uint64_t)1 << 32) + (uint64_t)p.mod - 1) / (uint64_t)p.mod) : 0xFFFFFFFFu;
  cudaStream_t st = G0->stream;
  ShardLink L = G0->link;
  L.lg = n;
  for (int i = 0; i < n; ++i) {
    prism_graph_t G = shards[i];
    G->recorded = 0;
    G->gathered_k = -1;
    const StateReq q{p.record ? (size_t)std::max<int64_t>(1, G->fin_rows) * Sp * 8 : 0, (size_t)P.G * Sp * 8,
                     (size_t)P.W * Sp * 8, 0, 0, 0, 0, 0};
    prism_status st = ensure_state(G, q);
    if (st) return st;
    L.lg_fin[i] = p.record ? G->fin : nullptr;
    L.lg_gfin[i] = G->gfin;
    L.lg_rank_end[i] = G->rank_end;
  }
  // every shard's earlier work (builds, overrides) is ordered before the launch on shard 0's stream
  std::vector<cudaEvent_t> evs;
  auto join = [&](cudaStream_t from, cudaStream_t to) -> cudaError_t {
    if (from == to) return cudaSuccess;
    cudaEvent_t e;
    cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (r != cudaSuccess) return r;
    evs.push_back(e);
    r = cudaEventRecord(e, from);
    return r == cudaSuccess ? cudaStreamWaitEvent(to, e, 0) : r;
  };
  for (int i = 1; i < n; ++i) CU(join(shards[i]->stream, st));
  CU(launch_replay_guard(G0->words, nullptr, 0, nullptr, 0, G0->parity, st));
  G0->rec(2);
  const int per_launch = cells_chunks_per_launch(G0->cur(), nchunks, n);
  int64_t launches = 1;
  for (int ch = 0; ch < nchunks; ch += per_launch) {
    CU(launch_cells(G0->cur(), p, nullptr, nullptr, nullptr, nullptr, G0->words, G0->parity, nullptr, nullptr, nullptr,
                    ch, std::min(per_launch, nchunks - ch), Sp, &L, st));
    ++launches;
  }
  for (int i = 0; i < n; ++i) {  // accumulators and counters of every shard's exchange buffer
    prism_graph_t G = shards[i];
    CU(cudaMemsetAsync(G->ex + G->link.o_acc, 0, (size_t)P.G_large * Sp * 8, st));
    CU(cudaMemsetAsync(G->ex + G->link.o_arrive, 0, (size_t)P.G_large * nchunks * 4, st));
    G->parity ^= 1;
  }
  G0->rec(3);
  G0->rec(4);
  CU(launch_local_group_reduce(G0->cur(), L, S, Sp, iter_dev, st));
  ++launches;
  G0->rec(5);
  CU(cudaMemcpyAsync(G0->h_status, G0->words, 8, cudaMemcpyDeviceToHost, st));
  for (int i = 1; i < n; ++i) CU(join(st, shards[i]->stream));
  for (cudaEvent_t e : evs) cudaEventDestroy(e);  // released once their work is done
  for (int i = 0; i < n; ++i) {
    prism_graph_t G = shards[i];
    G->last = p;
    G->last_Sp = Sp;
    G->recorded = p.record;
    G->last_algo = PRISM_ALGO_CELLS;
    G->launches = launches;
  }
  return PRISM_OK;
}

prism_status prism_shard_gather(prism_graph_t G, int32_t scenario) {
  if (!G) return fail(PRISM_E_INVALID_ARG, "null graph");
  if (G->n_shards < 2 || !G->connected || !G->ex) return fail(PRISM_E_INVALID_ARG, "not a connected shard");
  if (G->local_group) return fail(PRISM_E_INVALID_ARG, "shards of one device gather together (prism_shard_gather_local)");
  if (!G->recorded) return fail(PRISM_E_NOT_REPLAYED, "no replay with record != 0 has run on this graph");
  if (scenario < 0 || scenario >= G->last.S) return fail(PRISM_E_INVALID_ARG, "scenario outside the last replay");
  CU(cudaSetDevice(G->device));
  ShardLink L = G->link;
  L.lg = 0;
  CU(cudaMemsetAsync(G->words, 0, 4, G->stream));
  CU(launch_gather(G->cur(), L, G->fin, G->gfin, G->last_Sp, scenario, ++G->gather_epoch, G->words, G->stream));
  CU(cudaMemcpyAsync(G->h_status, G->words, 8, cudaMemcpyDeviceToHost, G->stream));
  CU(cudaStreamSynchronize(G->stream));
  prism_status st = check_status(G);
  if (st) return st;
  G->gathered_k = scenario;
  return PRISM_OK;
}

prism_status prism_shard_gather_local(const prism_graph_t *shards, int32_t n, int32_t scenario) {
  if (!shards || n < 2 || n > kMaxShards) return fail(PRISM_E_INVALID_ARG, "bad arguments");
  prism_graph_t G0 = shards[0];
  for (int i = 0; i < n; ++i) {
    const prism_graph_t G = shards[i];
    if (!G || G->n_shards != n || G->shard != i || !G->local_group || !G->recorded || G->device != G0->device ||
        G->last_Sp != G0->last_Sp || scenario < 0 || scenario >= G->last.S)
      return fail(PRISM_E_INVALID_ARG, "shard " + std::to_string(i) + " is not a recorded local shard of this group");
  }
  CU(cudaSetDevice(G0->device));
  ShardLink L = G0->link;
  L.lg = n;
  for (int i = 0; i < n; ++i) {
    L.lg_fin[i] = shards[i]->fin;
    L.lg_gfin[i] = shards[i]->gfin;
  }
  for (int i = 1; i < n; ++i) CU(cudaStreamSynchronize(shards[i]->stream));
  CU(launch_gather(G0->cur(), L, nullptr, nullptr, G0->last_Sp, scenario, 0, G0->words, G0->stream));
  CU(cudaStreamSynchronize(G0->stream));
  for (int i = 0; i < n; ++i) shards[i]->gathered_k = scenario;
  return PRISM_OK;
}

prism_status prism_shard_prepare(prism_graph_t G, int32_t n_scenarios, void *handle_out) {
  if (!G || !handle_out) return fail(PRISM_E_INVALID_ARG, "null argument");
  if (G->n_shards < 2) return fail(PRISM_E_INVALID_ARG, "graph was not built with n_shards > 1");
  if (n_scenarios < 1 || n_scenarios > (1 << 20)) return fail(PRISM_E_INVALID_ARG, "scenario count out of range");
  CU(cudaSetDevice(G->device));
  CU(cudaStreamSynchronize(G->stream));
  const Plan &P = G->plan;
  const int SCn = cells_chunk_scenarios();
  const int nchunks = (n_scenarios + SCn - 1) / SCn;
  const int64_t Sp = (int64_t)nchunks * SCn;
  size_t off = 0;
  auto carve = [&off](size_t bytes) {
    off = (off + 255) & ~(size_t)255;
    const size_t o = off;
    off += std::max<size_t>(bytes, 8);
    return o;
  };
  ShardLink L{};
  L.n = G->n_shards;
  L.self = G->shard;
  L.o_rslot = (int64_t)carve((size_t)P.M_cross * Sp * 8);
  L.o_acc = (int64_t)carve((size_t)P.G_large * Sp * 8);
  L.o_arrive = (int64_t)carve((size_t)P.G_large * nchunks * 4);
  L.o_part = (int64_t)carve((size_t)2 * G->n_shards * Sp * 8);
  L.o_flag = (int64_t)carve((size_t)G->n_shards * 4);
  L.o_gcol = (int64_t)carve((size_t)P.N * 8);
  L.o_ggcol = (int64_t)carve((size_t)P.G * 8);
  L.o_gflag = (int64_t)carve((size_t)G->n_shards * 4);
  const size_t bytes = off;
  for (void *p : G->ipc_open) cudaIpcCloseMemHandle(p);
  G->ipc_open.clear();
  if (G->ex) cudaFree(G->ex);
  G->ex = nullptr;
  G->connected = false;
  CU(cudaMalloc((void **)&G->ex, bytes));
  G->ex_bytes = bytes;
  CU(cudaMemset(G->ex, 0, bytes));
  CU(cudaMemset(G->ex + L.o_rslot, 0xFF, (size_t)P.M_cross * Sp * 8));  // "not yet" under parity 0
  CU(cudaDeviceSynchronize());
  G->parity = 0;
  G->gather_epoch = 0;
  G->gathered_k = -1;
  G->ex_S = n_scenarios;
  G->ex_Sp = (int32_t)Sp;
  G->link = L;
  cudaIpcMemHandle_t h;
  static_assert(sizeof(cudaIpcMemHandle_t) <= PRISM_SHARD_HANDLE_BYTES, "IPC handle size");
  std::memset(handle_out, 0, PRISM_SHARD_HANDLE_BYTES);
  if (cudaIpcGetMemHandle(&h, G->ex) == cudaSuccess) std::memcpy(handle_out, &h, sizeof h);
  else cudaGetLastError();  // IPC unavailable: only prism_shard_connect_local can be used
  return PRISM_OK;
}

prism_status prism_shard_connect(prism_graph_t G, const void *handles) {
  if (!G || !handles) return fail(PRISM_E_INVALID_ARG, "null argument");
  if (!G->ex) return fail(PRISM_E_INVALID_ARG, "call prism_shard_prepare first");
  CU(cudaSetDevice(G->device));
  const unsigned char *hb = (const unsigned char *)handles;
  for (int m = 0; m < G->n_shards; ++m) {
    if (m == G->shard) {
      G->link.base[m] = G->ex;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hb + (size_t)m * PRISM_SHARD_HANDLE_BYTES, sizeof h);
    void *p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(PRISM_E_CUDA, "cudaIpcOpenMemHandle of shard " + std::to_string(m) + ": " + cudaGetErrorString(e));
    }
    G->ipc_open.push_back(p);
    G->link.base[m] = (unsigned char *)p;
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.device == G->device &&
        !std::getenv("PRISM_ALLOW_SAME_DEVICE_IPC"))
      return fail(PRISM_E_INVALID_ARG, "shard " + std::to_string(m) + " lives on this process's device: separate "
                                       "processes' replays of one GPU are not guaranteed to run concurrently (set "
                                       "PRISM_ALLOW_SAME_DEVICE_IPC=1 for experiments; use one process per GPU)");
    cudaGetLastError();
  }
  G->local_group = false;
  G->connected = true;
  return PRISM_OK;
}

prism_status prism_shard_connect_local(prism_graph_t G, const prism_graph_t *shards) {
  if (!G || !shards) return fail(PRISM_E_INVALID_ARG, "null argument");
  if (!G->ex) return fail(PRISM_E_INVALID_ARG, "call prism_shard_prepare first");
  CU(cudaSetDevice(G->device));
  for (int m = 0; m < G->n_shards; ++m) {
    const prism_graph_s *o = shards[m];
    if (!o || !o->ex || o->n_shards != G->n_shards || o->shard != m || o->ex_bytes != G->ex_bytes)
      return fail(PRISM_E_INVALID_ARG, "shard " + std::to_string(m) + " is not a prepared peer of this graph");
    if (o->device != G->device) {
      int can = 0;
      CU(cudaDeviceCanAccessPeer(&can, G->device, o->device));
      if (!can) return fail(PRISM_E_CUDA, "no peer access between devices");
      cudaError_t e = cudaDeviceEnablePeerAccess(o->device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(PRISM_E_CUDA, cudaGetErrorString(e));
      cudaGetLastError();
    }
    G->link.base[m] = o->ex;
  }
  bool same = false;
  for (int m = 0; m < G->n_shards; ++m) same |= m != G->shard && shards[m]->device == G->device;
  G->local_group = same;
  G->connected = true;
  return PRISM_OK;
}

prism_status prism_shard_adopt(prism_graph_t G, prism_graph_t from) {
  if (!G || !from) return fail(PRISM_E_INVALID_ARG, "null argument");
  if (G == from) return PRISM_OK;
  const Plan &a = G->plan, &b = from->plan;
  if (!from->ex || !from->connected || G->n_shards != from->n_shards || G->shard != from->shard ||
      G->device != from->device || a.M_cross != b.M_cross || a.G_large != b.G_large || a.W != b.W)
    return fail(PRISM_E_INVALID_ARG, "adopt: `from` must be a connected shard graph of the same plan and shard");
  CU(cudaSetDevice(G->device));
  if (from->stream != G->stream) CU(cudaStreamSynchronize(from->stream));  // same stream: ordered
  for (void *p : G->ipc_open) cudaIpcCloseMemHandle(p);
  if (G->ex) cudaFree(G->ex);
  G->ex = from->ex;
  G->ex_bytes = from->ex_bytes;
  G->ex_S = from->ex_S;
  G->ex_Sp = from->ex_Sp;
  G->link = from->link;
  G->parity = from->parity;
  G->ipc_open = std::move(from->ipc_open);
  G->local_group = from->local_group;
  G->connected = true;
  from->ex = nullptr;
  from->ipc_open.clear();
  from->connected = false;
  return PRISM_OK;
}

prism_status prism_shard_info(prism_graph_t G, int32_t out[4]) {
  if (!G || !out) return fail(PRISM_E_INVALID_ARG, "null argument");
  out[0] = G->n_shards;
  out[1] = G->shard;
  out[2] = G->dg.shard_axis;
  out[3] = G->n_shards > 1 ? (G->dg.shard_axis == 1 ? G->plan.topo.pp : G->plan.topo.dp) / G->n_shards : 0;
  return PRISM_OK;
}

prism_status prism_graph_stats(prism_graph_t G, int64_t out[10]) {
  if (!G || !out) return fail(PRISM_E_INVALID_ARG, "null argument");
  const Plan &P = G->plan;
  out[0] = P.W;
  out[1] = P.N;
  out[2] = P.G;
  out[3] = P.M;
  out[4] = P.levels;
  out[5] = (int64_t)P.q.size();
  out[6] = P.sync_nodes;
  out[7] = P.max_group;
  out[8] = G->structure_bytes;
  out[9] = G->launches;
  return PRISM_OK;
}

prism_status prism_last_algo(prism_graph_t G, int32_t *algo_out) {
  if (!G || !algo_out) return fail(PRISM_E_INVALID_ARG, "null argument");
  *algo_out = G->last_algo;
  return PRISM_OK;
}

void prism_destroy_graph(prism_graph_t G) { delete G; }

prism_status prism_last_timing(prism_graph_t G, float out[5]) {
  if (!G || !out) return fail(PRISM_E_INVALID_ARG, "null argument");
  if (!G->profile) return fail(PRISM_E_INVALID_ARG, "graph was not built with PRISM_BUILD_PROFILE");
  CU(cudaSetDevice(G->device));
  const int pairs[5][2] = {{0, 1}, {2, 3}, {3, 4}, {4, 5}, {6, 7}};
  for (int i = 0; i < 5; ++i) {
    out[i] = -1.f;
    if (G->ev_done[pairs[i][0]] && G->ev_done[pairs[i][1]]) {
      CU(cudaEventSynchronize(G->ev[pairs[i][1]]));
      CU(cudaEventElapsedTime(&out[i], G->ev[pairs[i][0]], G->ev[pairs[i][1]]));
    }
  }
  return PRISM_OK;
}

}  // extern "C"

// ---- debug export (tests): copy device CSR arrays to host ------------------------------------
extern "C" PRISM_API prism_status prism_debug_export(prism_graph_t G, int32_t which, void *host_out, int64_t bytes) {
  if (!G || !host_out) return fail(PRISM_E_INVALID_ARG, "null argument");
  const DevGraph &d = G->dg;
  const void *src = nullptr;
  int64_t need = 0;
  switch (which) {
    case 0: src = d.rank_ptr; need = (d.W + 1) * 4; break;
    case 1: src = d.node_rank; need = d.N * 4; break;
    case 2: need = d.N * 8; break;  // 2-6: template fields, materialised below
    case 3: need = d.N; break;
    case 4: need = d.N * 4; break;
    case 5: need = d.N * 8; break;
    case 6: need = d.N * 8; break;
    case 7: src = d.node_prev_sync; need = d.N * 4; break;
    case 8: src = d.node_gptr; need = (d.N + 1) * 4; break;
    case 9: src = d.node_grp; need = d.M * 4; break;
    case 10: src = d.grp_ptr; need = (d.G + 1) * 4; break;
    case 11: src = d.grp_mem; need = d.M * 4; break;
    case 12: src = d.grp_dur; need = d.G * 8; break;
    case 13: src = d.grp_uid; need = d.G * 8; break;
    case 14: src = d.grp_level; need = d.G * 4; break;
    case 15: src = G->fin; need = G->recorded ? G->fin_rows * (int64_t)G->last_Sp * 8 : 0; break;
    default: return fail(PRISM_E_INVALID_ARG, "unknown array");
  }
  if (bytes < need) return fail(PRISM_E_INVALID_ARG, "buffer too small: need " + std::to_string(need));
  if (need == 0) return PRISM_OK;
  CU(cudaSetDevice(G->device));
  if (which >= 2 && which <= 6) {
    if (!G->ensure(G->scratch, G->scratch_bytes, (size_t)need)) return fail(PRISM_E_OOM, "scratch allocation failed");
    CU(launch_materialize(d, which, G->scratch, G->stream));
    src = G->scratch;
  }
  if (which == 15) {  // fin: device layout (graph.h fin_off) -> canonical [row = node][Sp], rank-major
    const int64_t rows = G->fin_rows, Sp = G->last_Sp, cw = Sp < 32 ? Sp : 32, n0 = G->fin_node0;
    std::vector<int64_t> raw((size_t)(rows * Sp));
    std::vector<int32_t> rp32((size_t)d.W + 1);
    CU(cudaMemcpyAsync(raw.data(), src, (size_t)need, cudaMemcpyDeviceToHost, G->stream));
    CU(cudaMemcpyAsync(rp32.data(), d.rank_ptr, (size_t)(d.W + 1) * 4, cudaMemcpyDeviceToHost, G->stream));
    CU(cudaStreamSynchronize(G->stream));
    int64_t *out = (int64_t *)host_out;
    const Plan &P = G->plan;
    for (int64_t r = 0; r < d.W; ++r) {
      // row of op 0 and row stride (graph.h cell_row0: TP cells, or replica cells with tp = 1)
      int64_t c0, stride;
      if (d.cell_R <= 1) {
        const int64_t tpi = r % d.tp;
        c0 = rp32[r - tpi] + tpi;
        stride = d.tp;
      } else {
        const int64_t R = d.cell_R;
        const bool meg = d.order == PRISM_ORDER_MEGATRON;
        const int64_t s2 = meg ? r / d.dp : r % d.pp, dpi = meg ? r % d.dp : r / d.pp;
        c0 = (meg ? (int64_t)d.dp * P.stage_op0[s2] + (dpi / R) * R * P.stage_len[s2]
                  : R * ((dpi / R) * d.Ltot + P.stage_op0[s2])) + dpi % R;
        stride = R;
      }
      for (int64_t n = rp32[r]; n < rp32[r + 1]; ++n) {
        if (n < n0 || n >= n0 + rows) continue;
        const int64_t row = c0 + (n - rp32[r]) * stride - n0;
        for (int64_t k = 0; k < Sp; ++k) out[(n - n0) * Sp + k] = raw[(size_t)(((k / cw) * rows + row) * cw + k % cw)];
      }
    }
    return PRISM_OK;
  }
  CU(cudaMemcpyAsync(host_out, src, (size_t)need, cudaMemcpyDeviceToHost, G->stream));
  CU(cudaStreamSynchronize(G->stream));
  return PRISM_OK;
}
