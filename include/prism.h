/*
 * prism.h — C ABI of the B200-native PrismLLM hot path (graph expansion + replay).
 *
 * What this library computes (PAPER.md = /root/reference/PAPER.md, "P:NNNN" = its line):
 *   - P:976-982 (§5.1, PrismTrace): the execution graph answers "what operations are executed,
 *     in what order, and how long"; nodes are compute spans or communication events with a
 *     duration; edges are *directional* ("one operation must complete before another begins")
 *     or *synchronization* ("all participating nodes must reach the operation before any can
 *     proceed (e.g., collectives or matched send-receive pairs)").
 *   - P:1099 (§5.2): "execution graphs are identical across DP groups" -> the input is a set of
 *     per-pipeline-stage op templates which prism_build_graph expands over TP/PP/DP/EP.
 *   - P:1295-1298 (§6.1): virtual ranks "wait for the recorded duration" at compute nodes and
 *     rendezvous at communication nodes -> prism_replay computes the ASAP schedule of every rank.
 *   - P:1573 (§8.1) iteration time = elapsed time of one step; P:1578 peak memory as
 *     max_memory_allocated -> prism_replay / prism_peak_memory.
 * Readings of silent points (Z1..Z16) are listed in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *   - Every call returns prism_status (0 = PRISM_OK). Nothing is thrown across the ABI.
 *     On error prism_last_error() returns a thread-local, human-readable detail string.
 *   - Every time is int64 nanoseconds, every size int64 bytes. No floating point on the path.
 *   - Input arrays are HOST pointers owned by the caller and copied during the call.
 *   - Output arrays are HOST pointers owned by the caller, unless the name says _dev.
 *   - A prism_graph owns its device buffers (allocated through prism_set_allocator's hooks,
 *     cudaMallocAsync if none) and releases them in prism_destroy_graph.
 *   - A graph handle is not thread-safe; distinct handles are independent.
 *   - All device work runs on the stream given at build time (prism_build_opts.stream).
 *   - There is no CPU fallback: without a CUDA device every compute call returns PRISM_E_CUDA.
 */
#ifndef PRISM_H
#define PRISM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRISM_ABI_VERSION 4

#if defined(__GNUC__)
#define PRISM_API __attribute__((visibility("default")))
#else
#define PRISM_API
#endif

typedef int32_t prism_status;
enum {
  PRISM_OK = 0,
  PRISM_E_INVALID_ARG = 1,       /* null pointer, size out of range, capacity too small       */
  PRISM_E_INVALID_SPEC = 2,      /* topology invalid: degrees < 1, ep does not divide dp, ... */
  PRISM_E_GA_TOO_SMALL = 3,      /* reserved (schedule generators)                */
  PRISM_E_TEMPLATE_MISMATCH = 4, /* a sync group is missing members or members disagree      */
  PRISM_E_DEADLOCK = 5,          /* the sync structure is cyclic: replay could never finish   */
  PRISM_E_NEGATIVE_MEMORY = 6,   /* a rank's running allocation would drop below zero        */
  PRISM_E_UNKNOWN_RANK = 7,      /* rank outside [0, world)                                   */
  PRISM_E_UNKNOWN_LABEL = 8,     /* reserved (what-if label overrides)                       */
  PRISM_E_NOT_REPLAYED = 9,      /* query before any prism_replay with record != 0            */
  PRISM_E_OOM = 10,              /* device allocation failed                                  */
  PRISM_E_CUDA = 11,             /* CUDA runtime error / no device                            */
  PRISM_E_NCCL = 12              /* cross-shard exchange failed                               */
};

/* Opaque graph handle; owns device buffers. */
typedef struct prism_graph_s *prism_graph_t;

/* ---- input format ------------------------------------------------------------------------ */

/* Node kinds ("a computation span or a communication event"). */
enum { PRISM_KIND_COMPUTE = 0, PRISM_KIND_COLLECTIVE = 1, PRISM_KIND_P2P = 2 };

/* Collective types (P:1444-1450 decomposition; informational except that all members of one
 * group must agree on it). */
enum { PRISM_COLL_AR = 0, PRISM_COLL_RS = 1, PRISM_COLL_AG = 2, PRISM_COLL_A2A = 3,
       PRISM_COLL_BCAST = 4, PRISM_COLL_BARRIER = 5 };

/* Communicator-group roles ("DP, TP, PP"; EP/EDP from the EP column of P:1983-1989).
 * The numeric values are also the role field of the group perturbation uid. */
enum { PRISM_ROLE_TP = 1, PRISM_ROLE_DP = 2, PRISM_ROLE_EP = 3, PRISM_ROLE_EDP = 4,
       PRISM_ROLE_WORLD = 5, PRISM_ROLE_P2P = 6 };

/* Batched point-to-point messages of one P2P node, between ring neighbours of the pipeline
 * (next = (stage+1) mod pp, prev = (stage-1) mod pp). The k-th SEND_NEXT of stage s pairs with
 * the k-th RECV_PREV of stage s+1 (same tp/dp coordinates); the k-th SEND_PREV of stage s pairs
 * with the k-th RECV_NEXT of stage s-1. Each message is a 2-member synchronization group
 * ("matched send-receive pairs"); a node with several messages finishes when all of them
 * have finished (reading Z3). */
enum { PRISM_P2P_SEND_NEXT = 1, PRISM_P2P_RECV_PREV = 2, PRISM_P2P_SEND_PREV = 4,
       PRISM_P2P_RECV_NEXT = 8 };

/* Rank numbering (reading Z1). TP_PP_DP: r = tp_i + tp*(pp_i + pp*dp_i) (TP fastest).
 * MEGATRON ("tp-cp-ep-dp-pp"): r = tp_i + tp*(dp_i + dp*pp_i). EP is carved out of DP:
 * ep_i = dp_i % ep, edp_i = dp_i / ep, in both orders. */
enum { PRISM_ORDER_TP_PP_DP = 0, PRISM_ORDER_MEGATRON = 1 };

typedef struct {
  int32_t tp, pp, dp, ep; /* world = tp*pp*dp; ep >= 1 divides dp                              */
  int32_t vpp;            /* informational (the schedule lives in the templates, reading Z16) */
  int32_t rank_order;     /* PRISM_ORDER_*                                                    */
} prism_topology;

/* One op of a per-stage template. 48 bytes, natural alignment, little-endian. */
typedef struct {
  uint8_t kind;      /* PRISM_KIND_*                                                          */
  uint8_t coll;      /* PRISM_COLL_* (COLLECTIVE only)                                        */
  uint8_t role;      /* PRISM_ROLE_TP..WORLD (COLLECTIVE only)                                */
  uint8_t p2p_mask;  /* PRISM_P2P_* bits, nonzero (P2P only)                                  */
  uint8_t stream;    /* 0..3: the rank's stream the op is issued on (row f2; 0 = single stream) */
  uint8_t ev_record; /* 0, or 1 + e: the op's finish records event slot e (e < 8)  (row f2)    */
  uint8_t ev_wait;   /* 0, or 1 + e: the op starts after the latest record of event slot e   */
  uint8_t pad0;
  uint32_t label;    /* user tag (queries / what-if); not interpreted                         */
  uint32_t pad1;
  int64_t dur_ns;    /* >= 0, <= 2^40. For sync ops: this member's duration of the occurrence */
  int64_t bytes;     /* payload, informational                                                */
  int64_t mem_alloc; /* >= 0: allocated at the op's start                                     */
  int64_t mem_free;  /* >= 0: freed at the op's finish                                        */
} prism_op;

typedef struct {
  const prism_op *ops;       /* concatenated templates, n_ops entries                          */
  int64_t n_ops;
  const int64_t *tmpl_ptr;   /* [pp+1]: stage s runs ops[tmpl_ptr[s] .. tmpl_ptr[s+1]) in order;
                                every rank of stage s runs the same template           */
  const int64_t *static_mem; /* [pp]: bytes resident for the whole iteration on stage-s ranks   */
} prism_templates;

/* Device-memory hooks (the Python binding routes these to PyTorch's caching allocator). */
typedef void *(*prism_alloc_fn)(size_t bytes, void *stream, void *ctx);
typedef void (*prism_free_fn)(void *ptr, void *stream, void *ctx);

typedef struct {
  void *stream;           /* cudaStream_t all device work of this graph is issued on (NULL = legacy
                             default stream)                                                  */
  int32_t device;         /* CUDA device ordinal, -1 = current                                 */
  int32_t n_shards;       /* >= 1: the replay is sharded over n_shards GPUs (row e; see the
                             "multi-GPU" section below); n_shards <= 16 divides dp or pp     */
  int32_t shard_index;    /* 0 .. n_shards-1: this shard replays the ranks of block shard_index
                             of the shard axis (DP blocks or PP-stage blocks, below)          */
  int32_t flags;          /* PRISM_BUILD_PROFILE: record CUDA events around every kernel group */
} prism_build_opts;

/* PRISM_BUILD_PROFILE: record CUDA events around every kernel group (prism_last_timing).
 * PRISM_BUILD_ASYNC: return once the expansion is queued on the stream (later calls on the same
 * stream are ordered after it); by default prism_build_graph waits for it.
 * PRISM_BUILD_SHARD_DP / _PP: force the shard axis of a sharded build (default: the axis whose
 * blocks cut the fewest exchanged synchronisations — template-level sync ops whose group spans
 * shards, chained collectives excepted — SURVEY §8.4; every shard resolves the same axis). */
enum { PRISM_BUILD_PROFILE = 1, PRISM_BUILD_ASYNC = 2, PRISM_BUILD_SHARD_DP = 4, PRISM_BUILD_SHARD_PP = 8 };

/* Scenario batch for what-if sweeps (re-time without structural change).
 * Scenario k gets perturbed durations d' = (d * (65536 + delta)) >> 16 with
 * delta = ((h >> 40) mod (2*amp+1)) - amp, h = splitmix64(seed ^ k*0x9E3779B97F4A7C15 ^
 * uid*0xBF58476D1CE4E5B9); uid = (rank<<32)|template_index for compute nodes and
 * (role<<56)|(gid<<24)|occurrence for sync groups (exact text in DESIGN.md §3, Z8).
 * Scenario 0, and every node kind whose bit (1<<kind) is clear in kind_mask, is unperturbed. */
typedef struct {
  int32_t n;          /* S >= 1 scenarios                                                     */
  int32_t amp_q16;    /* 0 .. 65535                                                           */
  uint64_t seed;
  uint32_t kind_mask; /* bit (1<<PRISM_KIND_*) = perturb that kind                             */
  int32_t record;     /* nonzero: keep every node's finish time for prism_query_rank           */
  int32_t algo;       /* PRISM_ALGO_AUTO (cells when they fit on the device, else levels),
                         PRISM_ALGO_LEVELS (one launch per frontier level), PRISM_ALGO_CELLS   */
  int32_t first;      /* global index of the batch's first scenario: local scenario j is
                         scenario first + j of the sweep (perturbation key k = first + j; only
                         global scenario 0 is unperturbed). Lets a sweep run in batches or be
                         split over GPUs; outputs stay indexed by the local j.                */
  int32_t pad;
} prism_scenarios;

/* PRISM_ALGO_RANKS: one scenario, one rank per lane (auto picks it for n == 1 when the graph is
 * unsharded and single-stream with tp a power of two <= 32). */
enum { PRISM_ALGO_AUTO = 0, PRISM_ALGO_LEVELS = 1, PRISM_ALGO_CELLS = 2, PRISM_ALGO_RANKS = 3 };

/* ---- entry points ------------------------------------------------------------------------ */

PRISM_API const char *prism_status_string(prism_status s);
PRISM_API const char *prism_last_error(void);
PRISM_API int32_t prism_abi_version(void);

/* Install device allocation hooks used by subsequent prism_build_graph calls (NULL, NULL =
 * cudaMallocAsync/cudaFreeAsync). Process-global; not thread-safe against concurrent builds. */
PRISM_API prism_status prism_set_allocator(prism_alloc_fn alloc, prism_free_fn free_fn, void *ctx);

/* Rows a1-a5: expand the per-stage templates over the topology into the device-resident CSR
 * DAG: node SoA (rank, duration, kind, label, alloc/free), per-node sync-group lists, sync-group
 * CSR (members, shared duration = max of members' dur_ns (Z2), perturbation uid, level) sorted
 * by level. Validates everything on the host before any launch:
 *   PRISM_E_INVALID_SPEC       bad topology
 *   PRISM_E_INVALID_ARG        malformed op (unknown kind/role, negative duration/bytes, stream!=0,
 *                              P2P with pp==1, empty p2p_mask, dur > 2^40), N or M >= 2^31
 *   PRISM_E_TEMPLATE_MISMATCH  a P2P message without its partner, WORLD collectives whose count or
 *                              collective type differ between stages
 *   PRISM_E_DEADLOCK           the synchronization structure has a cycle
 *   PRISM_E_NEGATIVE_MEMORY    a template's running allocation drops below zero (program order)
 * On success *out owns the graph. Blocks until the device work is complete unless
 * opts.flags has PRISM_BUILD_ASYNC. Host plan cache: a build whose topology, template arrays
 * (ops, tmpl_ptr, static_mem, compared byte for byte) and shard options (n_shards, shard_index,
 * flags) equal one of the last four successful builds' reuses that build's validated plan instead
 * of planning again (same result; the environment variable PRISM_PLAN_CACHE=0 disables it). */
PRISM_API prism_status prism_build_graph(const prism_topology *topo, const prism_templates *tmpl,
                               const prism_build_opts *opts, prism_graph_t *out);

/* Host-only dry run of prism_build_graph's validation and quotient plan (no device needed):
 * out[0..7] = world, nodes, sync groups, memberships, levels, quotient groups, sync nodes,
 * max group size. Same error statuses as prism_build_graph. */
PRISM_API prism_status prism_plan(const prism_topology *topo, const prism_templates *tmpl, int64_t out[8]);

/* Rows a6-a8: replay all ranks over the graph for S scenarios (ASAP, integer ns, reading Z4/Z5):
 * a compute node starts when its stream predecessor finishes; a sync group starts at the max of
 * its members' ready times (segmented max) and lasts its (perturbed) duration; a sync node
 * finishes at the max over its groups. Writes the iteration time T_k = max finish (ns) of each
 * scenario to iter_ns_out[k] (host, n entries). Synchronizes the stream. */
PRISM_API prism_status prism_replay(prism_graph_t g, const prism_scenarios *sc, int64_t *iter_ns_out);

/* Same as prism_replay but asynchronous: writes T_k into iter_ns_dev_out (DEVICE pointer, n
 * int64) on the graph's stream and returns without synchronizing. The returned status covers the
 * host-side checks only; whether the device finished the replay is reported by the next
 * synchronizing call on the graph (prism_sync, prism_replay, prism_query_rank, ...): if a replay
 * queued since the last such call was aborted by the device watchdog, that call returns
 * PRISM_E_DEADLOCK once, and the iteration times of those replays are invalid. */
PRISM_API prism_status prism_replay_async(prism_graph_t g, const prism_scenarios *sc, int64_t *iter_ns_dev_out);

/* Waits for every call queued on the graph's stream and reports what the device found since the
 * last synchronizing call: PRISM_E_DEADLOCK if a replay was aborted by the device watchdog (a
 * waiting warp saw no progress for the watchdog period, 10 s by default), PRISM_E_NEGATIVE_MEMORY
 * if a time-ordered memory scan found a negative running total; PRISM_OK otherwise. After an
 * abort the next replay of an unsharded graph first resets its ready slots (bit-exact results
 * again); a sharded graph must be re-prepared (prism_shard_prepare / _connect). */
PRISM_API prism_status prism_sync(prism_graph_t g);

/* Row a9: per-rank peak memory in bytes, peak_r = static_mem[stage(r)] + max(0, max prefix sum of
 * the rank's events +alloc at op start / -free at op finish ordered by (time, event index)); for
 * single-stream ranks this is program order (Z6), so the result does not depend on
 * the scenario and no replay is required. Writes world entries to peak_bytes_out (host). */
PRISM_API prism_status prism_peak_memory(prism_graph_t g, int64_t *peak_bytes_out);
PRISM_API prism_status prism_peak_memory_async(prism_graph_t g, int64_t *peak_bytes_dev_out);

/* Row f2 (multi-stream ranks): per-rank peak memory with the events in TIME order, (time, event
 * index), of scenario `scenario` of the last recorded replay (the starts and finishes the replay
 * computed). For single-stream graphs this equals prism_peak_memory (program order = time order,
 * reading Z6); prism_peak_memory / _async of a multi-stream graph compute it for scenario 0.
 * PRISM_E_NOT_REPLAYED without a recorded replay; PRISM_E_NEGATIVE_MEMORY if a running total
 * drops below zero in time order; PRISM_E_INVALID_ARG beyond 4096 ops per rank, or on a sharded
 * graph whose scenario was not gathered (prism_shard_gather). */
PRISM_API prism_status prism_peak_memory_at(prism_graph_t g, int32_t scenario, int64_t *peak_bytes_out);

/* ---- multi-GPU (row e): rank sharding with a fused peer-memory exchange ---------------------
 *
 * The ranks are partitioned into n blocks along one axis (north_star: "Ranks are sharded across
 * the 8 B200s of one box"): DP blocks (shard i owns every rank whose dp coordinate lies in
 * [i*dp/n, (i+1)*dp/n); TP groups and P2P messages stay inside a block, DP / EP / EDP / WORLD
 * collectives may span shards) or PP-stage blocks (pp coordinate in [i*pp/n, (i+1)*pp/n); every
 * collective but WORLD stays inside a block, P2P messages at block edges span shards; SURVEY §8(e)
 * picks these for the MoE config, whose EP all-to-alls would otherwise all cross shards).
 * Every shard holds the whole (replicated, O(N)) graph structure and replays only its own cells;
 * the cell kernel pushes the ready time of a member of a cross-shard group straight into the
 * exchange buffer of every shard holding a member of that group (NVLink peer stores and red.max
 * atomics at system scope) and polls its local copy, so the segmented max over a group's members
 * ("all participating nodes must reach the operation before any can proceed") is done by the
 * replay kernel itself, tile by tile, instead of by a separate collective between launches. The
 * iteration time is the max over shards of each shard's partial max, exchanged the same way by the
 * final reduce kernel, so every shard returns the same T_k. Results are bit-identical to n = 1.
 *
 * Protocol (SPMD, every shard calls the same functions in the same order):
 *   1. prism_build_graph with opts.n_shards = n, opts.shard_index = i on the shard's device;
 *   2. prism_shard_prepare(g, S, handle): allocates the shard's exchange buffer for replays of
 *      exactly S scenarios and writes its CUDA IPC handle (PRISM_SHARD_HANDLE_BYTES bytes);
 *   3. all-gather the n handles (the Python binding uses torch.distributed), then
 *      prism_shard_connect(g, handles[n]) opens the peers' buffers; or, when all shards live in
 *      one process, prism_shard_connect_local(g, graphs[n]);
 *   4. prism_replay / prism_replay_async with n == S on every shard (one process per GPU); the
 *      replays of all shards run concurrently, since a shard's kernel waits for its peers' ready
 *      times; a shard that never arrives is reported by the device watchdog as PRISM_E_DEADLOCK
 *      (10 s) instead of hanging the GPU. Shards sharing one device replay together through
 *      prism_replay_local_shards.
 * prism_peak_memory returns all world peaks on every shard (the structure is replicated);
 * prism_query_rank answers for the shard's own ranks (PRISM_E_INVALID_ARG names the owner
 * otherwise) and, after prism_shard_gather of the scenario, for every rank. Replaying a sharded graph before connect, or with n != S, is PRISM_E_INVALID_ARG.
 * The exchange buffer is released with the graph; peers must destroy their graphs only after the
 * last replay of every shard has completed. */
#define PRISM_SHARD_HANDLE_BYTES 64

/* Per-rank outputs of a sharded replay gathered to every shard ("per-rank outputs
 * are gathered to each caller"): collective over the shards (SPMD, every shard calls it after the
 * same replay), it copies every shard's recorded finish times of scenario `scenario` into every
 * shard's gather columns over NVLink peer stores (epoch-flag barrier, device watchdog). Until the
 * next replay, prism_query_rank (any rank), prism_critical_path and prism_peak_memory_at answer
 * that scenario on every shard; other scenarios stay owner-only / PRISM_E_INVALID_ARG.
 * Synchronizes the stream. Shards of one device gather together: prism_shard_gather_local. */
PRISM_API prism_status prism_shard_gather(prism_graph_t g, int32_t scenario);
PRISM_API prism_status prism_shard_gather_local(const prism_graph_t *shards, int32_t n, int32_t scenario);
/* out[0..3] = n_shards, shard index, shard axis (0 = DP blocks, 1 = PP-stage blocks), block size
 * (dp or pp coordinates per shard; 0 unsharded). */
PRISM_API prism_status prism_shard_info(prism_graph_t g, int32_t out[4]);
PRISM_API prism_status prism_shard_prepare(prism_graph_t g, int32_t n_scenarios, void *handle_out);
PRISM_API prism_status prism_shard_connect(prism_graph_t g, const void *handles);
PRISM_API prism_status prism_shard_connect_local(prism_graph_t g, const prism_graph_t *shards);
/* Shards living on ONE device (connected with prism_shard_connect_local) cannot rely on separate
 * launches running concurrently (CUDA does not guarantee it; profilers and MPS serialise them),
 * so they replay together: one cooperative launch covers every shard's cells (co-residency is
 * checked before the launch), the exchange between shards runs through the same peer-memory
 * protocol, and one reduce writes T_k (n int64, DEVICE pointer) on shards[0]'s stream, ordered
 * after and before the other shards' streams. Every shard records its own ranks' times (query
 * them on the owning shard). The shards must carry the same duration overrides (the launch reads
 * shards[0]'s graph structure). prism_replay / _async on such a shard return PRISM_E_INVALID_ARG,
 * as does prism_shard_connect when a peer's buffer is on the caller's own device. */
PRISM_API prism_status prism_replay_local_shards(const prism_graph_t *shards, int32_t n, const prism_scenarios *sc,
                                                 int64_t *iter_ns_dev_out);
/* Move the connected exchange buffer (and the peers' mapping of it) of `from` to a newly built
 * graph g of the same plan and shard (a rebuilt graph keeps its communicator; SPMD: every shard
 * adopts at the same point of its call sequence). Waits for `from`'s stream unless both graphs
 * use the same stream (then stream order suffices); `from` is left unconnected. PRISM_E_INVALID_ARG if the plans' exchange layouts or the shards differ. */
PRISM_API prism_status prism_shard_adopt(prism_graph_t g, prism_graph_t from);

/* ---- rows f1 / f3 / f4: per-node durations, memory deltas, critical path -------------------
 *
 * f1, inter-slice calibration (§5.3): "timing within each slice is locally accurate
 * but not globally aligned"; the timed graph (one measured duration per node, each rank measured
 * in the slice where it ran as a real rank) is re-timed by the same ASAP replay, which shifts a
 * receive after its send and propagates (node_dur).
 * f3, what-if attribution ("a fake GPU kernel that spins for the desired and
 * optimized duration"): label overrides, per-rank compute slowdown (fault
 * injection) and the critical path (prism_critical_path).
 * f4, MoE imbalance (P:1745-1748 mock router; App. F): prism_set_moe_load below.
 * Effective duration of node n (node order = rank-major, program order, as prism_query_rank):
 *   d = node_dur ? node_dur[n] : template dur_ns;  d = (d * br) >> 16 if the node's template op is
 *   routed (prism_set_moe_load);  d = label_dur[i] if label(n) == labels[i];
 *   d = (d * rank_slow_q16[rank(n)]) >> 16 if node n is a compute span.
 * A synchronization group lasts the max of its members' effective durations (reading Z2), and
 * scenario perturbation (prism_scenarios) applies on top. Arrays are copied: node_dur, node_alloc
 * and node_free may be host or device pointers (unified addressing; measured durations already on
 * the GPU are copied device to device), the label arrays and rank_slow_q16 are host. Applies to all
 * later replays / peak scans until reset with d == NULL (or all fields empty); invalidates the
 * recorded replay. Errors: PRISM_E_INVALID_ARG (duration outside [0, 2^40], memory delta outside
 * [0, 2^43], factor outside [0, 2^20], duplicate label), PRISM_E_UNKNOWN_LABEL (no node carries a
 * label), PRISM_E_NEGATIVE_MEMORY (a rank's running allocation would drop below zero in
 * program order). Per-node values are validated on the device; a failed call leaves the graph's
 * previous overrides in place. Synchronizes the stream. */
typedef struct {
  const int64_t *node_dur;       /* [N] or NULL                                                  */
  const uint32_t *labels;        /* [n_labels] label overrides ...                               */
  const int64_t *label_dur;      /* [n_labels] ... and their durations                           */
  int32_t n_labels;
  int32_t pad;
  const int32_t *rank_slow_q16;  /* [world] or NULL: compute-span factor, Q16 (65536 = 1.0)      */
  const int64_t *node_alloc;     /* [N] or NULL: bytes allocated at the node's start             */
  const int64_t *node_free;      /* [N] or NULL: bytes freed at the node's finish                */
} prism_durations;

PRISM_API prism_status prism_set_durations(prism_graph_t g, const prism_durations *d);

/* Row f4, MoE imbalance: the mock router of App. F ("The br represents the ratio of the
 * actual data volume possessed by a specific rank to the volume it would possess under a
 * perfectly uniform distribution ... multiple gating operations occur, each requiring control
 * via br"). Gating event v is one routing decision (one per MoE layer and microbatch, reading R7);
 * br_q16[v * ep + e] is the balance ratio of EP rank e in event v, Q16 (65536 = the uniform share).
 * Every node running a template op i with op_event[i] = v >= 0 on a rank with EP coordinate e
 * processes br times the uniform volume, so (scale bits) its duration, its allocation at start and
 * its free at finish are scaled: x' = (x * br_q16[v * ep + e]) >> 16 (floor). A routed all-to-all's
 * members then last different times and the group lasts their max (reading Z2). Applied on top of
 * prism_set_durations' base values (measured, else template) and before its label overrides and
 * rank slowdown; both calls compose. m == NULL or m->n_events == 0 clears the load.
 * Arrays are host, copied: op_event [n_ops of the templates] in [-1, n_events), br_q16
 * [n_events][ep] in [0, 2^20]. Errors: PRISM_E_INVALID_ARG (out-of-range entries, unknown scale
 * bits), PRISM_E_NEGATIVE_MEMORY (scaled allocations and frees that drive a rank's running
 * allocation below zero). Invalidates the recorded replay; synchronizes the stream. */
enum { PRISM_MOE_DUR = 1, PRISM_MOE_ALLOC = 2, PRISM_MOE_FREE = 4 };
typedef struct {
  const int32_t *op_event;  /* [n_ops] gating event of each template op, -1 = not routed        */
  const int32_t *br_q16;    /* [n_events][ep] balance ratios, Q16                                */
  int32_t n_events;
  uint32_t scale;           /* PRISM_MOE_* bits: which of duration / alloc / free scale with br  */
} prism_moe_load;

PRISM_API prism_status prism_set_moe_load(prism_graph_t g, const prism_moe_load *m);

/* Row f3: the critical path of scenario `scenario` of the last recorded replay, walked back from
 * the lowest-numbered node finishing at T: a compute span continues at its stream predecessor; a
 * synchronization node at the group with the max (start + duration') among its groups (lowest uid
 * on ties), then at the stream predecessor of that group's latest-ready member (lowest node id on
 * ties); the walk ends at a node with no predecessor edge. path_out[0..n) = the nodes, last first;
 * *T_out = T. If cap < n: *n_out = n and PRISM_E_INVALID_ARG. PRISM_E_NOT_REPLAYED without a
 * recorded replay; sharded graphs are not supported (PRISM_E_INVALID_ARG). */
PRISM_API prism_status prism_critical_path(prism_graph_t g, int32_t scenario, int32_t *path_out, int64_t cap,
                                           int64_t *n_out, int64_t *T_out);

/* Per-op start and finish times of one rank in one scenario of the last recorded replay, in
 * program order, plus the rank's coordinates (tp, pp, dp, ep, edp). If cap < the rank's op count
 * the call writes the count to *n_ops_out and returns PRISM_E_INVALID_ARG.
 * PRISM_E_NOT_REPLAYED if no replay with record != 0 has run; PRISM_E_UNKNOWN_RANK. */
PRISM_API prism_status prism_query_rank(prism_graph_t g, int32_t rank, int32_t scenario, int64_t *start_ns,
                              int64_t *finish_ns, int64_t cap, int64_t *n_ops_out,
                              int32_t coords_out[5]);

/* out[0..9]: world, nodes, sync groups, memberships, levels, quotient groups, sync nodes,
 * max group size, bytes of device graph structure, replay launches per call. */
PRISM_API prism_status prism_graph_stats(prism_graph_t g, int64_t out[10]);

/* Releases the graph. Device buffers are freed in stream order (no host wait) unless the graph
 * is a connected shard (its exchange buffer is synchronously released). */
PRISM_API void prism_destroy_graph(prism_graph_t g);

/* Schedule used by the last replay: PRISM_ALGO_LEVELS, _CELLS or _RANKS (0 before any). */
PRISM_API prism_status prism_last_algo(prism_graph_t g, int32_t *algo_out);

/* Device time (ms, CUDA events on the graph's stream) of the last call of each kernel group of a
 * graph built with PRISM_BUILD_PROFILE: out[0] expand (a1-a4, last build), out[1] level loop of the
 * last replay (a5-a7), out[2] tail (a6), out[3] iteration reduce (a8), out[4] peak scan (a9).
 * Synchronizes on the recorded events. PRISM_E_INVALID_ARG if profiling is off. */
PRISM_API prism_status prism_last_timing(prism_graph_t g, float out[5]);

/* Test hooks of the device watchdog: PRISM_DEBUG_WATCHDOG_NS sets the period after which a
 * waiting replay kernel aborts with PRISM_E_DEADLOCK (default 10 s, >= 1000); PRISM_DEBUG_STALL_UNIT
 * >= 0 makes that warp (cell kernel unit / rank kernel warp) of the following replays return at
 * once without arriving anywhere, so its partners time out (-1 = off). */
enum { PRISM_DEBUG_WATCHDOG_NS = 0, PRISM_DEBUG_STALL_UNIT = 1 };
PRISM_API prism_status prism_debug_set(prism_graph_t g, int32_t key, int64_t value);

/* Test hook: copy one device array of the graph to host memory (bytes = capacity of host_out).
 * which: 0 rank_ptr[W+1] i32, 1 node_rank[N] i32, 2 node_dur[N] i64, 3 node_kind[N] u8,
 * 4 node_label[N] u32, 5 node_alloc[N] i64, 6 node_free[N] i64, 7 node_prev_sync[N] i32,
 * 8 node_gptr[N+1] i32, 9 node_grp[M] i32, 10 grp_ptr[G+1] i32, 11 grp_mem[M] i32,
 * 12 grp_dur[G] i64, 13 grp_uid[G] u64, 14 grp_level[G] i32, 15 fin[N][S_pad] i64 (last
 * recorded replay; S_pad = S rounded up to the replay's scenario chunk). */
PRISM_API prism_status prism_debug_export(prism_graph_t g, int32_t which, void *host_out, int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* PRISM_H */
