// prism_internal.h — shared declarations of the CUDA path (kernels + C ABI). Not part of the ABI.
//
// Data layout in HBM:
//   node SoA, rank-major / program order:  node_rank[N] i32, node_dur[N] i64, node_kind[N] u8,
//     node_label[N] u32, node_alloc[N] i64, node_free[N] i64, node_prev_sync[N] i32 (previous
//     sync node of the same rank, -1 if none), node_gptr[N+1] i32 -> node_grp[M] i32 (the sync
//     groups of a node, slot order = P2P mask bit order).
//   sync-group CSR sorted by level:  grp_ptr[G+1] i32 -> grp_mem[M] i32 (member node ids),
//     grp_dur[G] i64 (max of members' op durations, reading Z2), grp_uid[G] u64 (perturbation
//     uid), grp_level[G] i32.
//   replay state (per call):  fin[N][S] i64 (scenario-fastest: one node's S finishes are one
//     contiguous 8*S-byte run), gfin[G][S] i64 (group finish = max member ready + dur'),
//     rank_end[W][S] i64, iter[S] i64.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/prism.h"

namespace prism {

// Cross-cell groups with at most this many members use the value-as-flag protocol of the cell
// kernel (ready slots); larger ones use max-accumulators + arrival counters.
constexpr int32_t kSmallGroup = 8;
// Row f2: streams per rank and CUDA-event slots of the template format.
constexpr int32_t kMaxStreams = 4;
constexpr int32_t kMaxEvents = 8;

// One quotient group: a template-level synchronization (all concrete instances are symmetric
// under the topology, so level / duration / member positions are per quotient group).
struct QGroup {
  int32_t type;        // PRISM_ROLE_TP..WORLD (collective) or PRISM_ROLE_P2P
  int32_t stage;       // collective: the stage of every member; P2P: sender stage
  int32_t tidx;        // collective: template index; P2P: sender template index
  int32_t slot;        // node_grp slot of the membership (sender for P2P)
  int32_t stage2;      // P2P receiver stage
  int32_t tidx2;       // P2P receiver template index
  int32_t slot2;       // P2P receiver slot
  int32_t size;        // members per concrete group
  int32_t inst;        // concrete instances
  int32_t level;       // 1-based frontier level
  int32_t occ;         // occurrence number (uid low bits)
  int32_t dir;         // P2P: 0 = SEND_NEXT/RECV_PREV, 1 = SEND_PREV/RECV_NEXT
  int32_t wpos;        // WORLD: offset of its per-stage template indices in the wpos table
  int32_t pad;
  int64_t dur;         // shared duration (max over member ops)
  int64_t gbase;       // first concrete group id
  int64_t mbase;       // first membership index
  int64_t xbase;       // first ready slot (cell kernel, small cross-cell groups); -1 otherwise
  int64_t lbase;       // first accumulator index (cell kernel, large groups); -1 otherwise
  // replica cells (Plan::cell_R > 1): a group holding all R replicas of a cell exchanges ONE value
  // per cell: cell-level ready slots (size / R <= kSmallGroup) or accumulator; -1 otherwise
  int64_t cxbase, clbase;
};

// A cross-cell op of a stage template: its template index, first slot offset and slot count;
// flags bit 0 (replica cells): the op's group holds every rank of the cell (one member per cell).
struct XOp {
  int32_t tidx, hoff, ns, flags;
};

struct Topo {
  int32_t tp, pp, dp, ep, order;
};

// Host-side plan of a graph (validation + quotient analysis), produced by plan_graph().
struct Plan {
  Topo topo;
  int64_t W = 0, N = 0, G = 0, M = 0, sync_nodes = 0;
  int64_t M_cross = 0;  // memberships of small cross-cell groups (cell-kernel ready slots)
  int64_t G_large = 0;  // cross-cell groups larger than kSmallGroup (cell-kernel accumulators)
  int32_t levels = 0, max_group = 0;
  // per template op (concatenated over stages, indexed by global op index)
  std::vector<int32_t> t_prev_sync;  // template-local index of the previous sync op, -1
  std::vector<int32_t> t_slot_ptr;   // template-local slot prefix (exclusive), per op
  std::vector<int32_t> t_slots;      // slots of each op
  std::vector<int64_t> stage_len;    // [pp]
  std::vector<int64_t> stage_slots;  // [pp] total slots per template
  // replay class of every template op (cell kernel): 0 compute span, 1 TP collective (the cell's
  // own group), 2 cross-cell synchronization, 3 chained collective: a DP/EP/EDP/WORLD collective
  // that immediately follows a collective of the same group, so every member is ready exactly at
  // that group's shared finish and start = own ready time (exact)
  std::vector<uint8_t> t_cls;
  std::vector<int32_t> t_q0;  // quotient group (index into q) of each template op's first slot, -1
  // row f2 (multi-stream ranks): any op off stream 0 or with an event; per template op the
  // previous op of its stream / the event source (template index, -1) and the packed
  // stream | ev_record << 4 | ev_wait << 8
  bool multistream = false;
  int32_t ms_streams = 0, ms_events = 0;  // streams used; distinct event slots (renumbered densely)
  std::vector<int32_t> t_spred, t_esrc;
  std::vector<uint16_t> t_ms;
  // per stage, the cross-cell ops (class 2) in template order: x_ptr[pp+1] -> XOp
  std::vector<int32_t> x_ptr;
  std::vector<XOp> x_ops;
  std::vector<int64_t> stage_op0;    // [pp] first global op index
  std::vector<QGroup> q;             // sorted by (level, creation order)
  std::vector<int32_t> wpos;         // WORLD template indices, pp per WORLD quotient group
  std::vector<int32_t> level_q_ptr;  // [levels+2]: quotient groups of level l = [ptr[l], ptr[l+1])
  // per template slot (stage-major; stage s's slots start at stage_slot0[s]): the quotient group
  // it joins (index into q), its template op, its member role in a P2P message (0 sender,
  // 1 receiver) and whether it is its op's first slot
  std::vector<int64_t> stage_slot0;  // [pp+1]
  std::vector<int32_t> slot_q, slot_tidx;
  std::vector<uint8_t> slot_role, slot_first;
  // group-side build chunks: (quotient group, first local membership), 2048 memberships each
  std::vector<int32_t> chunk_q;
  std::vector<int64_t> chunk_m;
  // replica cells (tp = 1): a cell of the cell kernel is cell_R consecutive DP replicas of one
  // stage instead of one TP group (1 = TP cells); per stage, the cell records of its cross ops
  // start at crec_ptr[s] (cells x cross ops of the stage)
  int32_t cell_R = 1;
  int32_t cta_ks = 1;  // EP CTAs: cells per CTA (1 = one warp per CTA)
  std::vector<int64_t> crec_ptr;
};

// Replica cells (row a6/a7): with tp = 1 the cell kernel's warps walk R consecutive
// DP replicas of a stage. A collective whose group holds all R replicas (DP, WORLD, EP when R
// divides ep, EDP when ep = 1) is reduced over the cell in registers and exchanged with ONE
// value per cell; a group holding one replica per cell (TP and EP of size 1, EDP when R divides
// ep, P2P messages) keeps its per-rank exchange. Rewrites the replay classes, marks the cell-full
// cross ops and allocates cell-level slots. Requires tp == 1, R | dp and (ep == 1 or R | ep).
// ks > 1 (EP CTAs): the ks cells of one EP group (ep = R ks) share a CTA, and an EP collective
// becomes class 4: the group's max is formed in registers and shared memory behind one CTA
// barrier, with no global exchange at all.
prism_status plan_replica_cells(Plan &P, int32_t R, int32_t ks, std::string &err);
bool replica_cells_ok(const Topo &t, int32_t R);

// Returns PRISM_OK or an error status with *err filled.
prism_status plan_graph(const prism_topology &topo, const prism_templates &tm, Plan &plan,
                        std::string &err);

// ---- device helpers -------------------------------------------------------------------------
#ifdef __CUDACC__
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
#endif

}  // namespace prism
