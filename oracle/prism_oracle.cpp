// prism_oracle.cpp — TEST INFRASTRUCTURE ONLY (the parity authority for the CUDA path).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
// load this library. It shares no code, header, table or helper with paper_2605_15617_b200/:
// the template record layout below is re-declared here from the input format (48-byte prism_op,
// written by workloads/), and every step is re-derived from the paper's definitions.
//
// What it computes, step by step (PAPER.md = /root/reference/PAPER.md):
//   1. Expansion (§5.2 "execution graphs are identical across DP groups"): every rank of
//      pipeline stage s runs template s; nodes are numbered rank-major in program order.
//   2. Communicator groups (§6.2 "DP, TP, PP" groups; EP/EDP from P:1983-1989): the k-th
//      collective of role R in a rank's template joins the k-th occurrence of the rank's
//      concrete R group; each P2P message is a 2-member "matched send-receive pair".
//   3. Replay (P:982 directional vs synchronization edges; "waits for the recorded
//      duration"; "shift the receive to occur after the send ... propagating"):
//      a discrete-event simulation with a min-heap of (time, node) finish events. A node is
//      released when its stream predecessor finishes; a compute node finishes dur' later; a
//      sync node arrives at each of its groups; when a group has all members, it starts at the
//      max of their arrival times and lasts its duration; a member finishes when all of its
//      groups have finished (max). Iteration time = max finish.
//      Row f2 (P:699, P:1729 overlapped communication): a rank issues its ops in template order
//      onto up to 4 streams; a node is released when the previous op of its stream AND (if it
//      waits on event slot e) the latest earlier op recording e have finished (CUDA-event
//      semantics; a wait on a never-recorded slot is satisfied at once).
//   4. Peak memory (P:1578 max_memory_allocated): per rank, events +alloc at op start and
//      -free at op finish sorted by (time, event index), prefix-summed; peak = static + max(0,
//      max prefix). A negative running total is an error.
// Readings of silent points are DESIGN.md §3 (Z1-Z16); the perturbation formula is Z8's text.
// Parity pins for this file: tests/test_oracle_pins.py (closed forms, brute force, hand-worked levels
// (tests/golden/levels_hand.txt), perturbation worked through SplitMix64's published outputs, SPEC worked
// examples, invariants).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <queue>
#include <string>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>

namespace {

struct Op {  // one template record, 48 bytes (input format)
  uint8_t kind, coll, role, p2p_mask, stream, ev_record, ev_wait, pad0;
  uint32_t label, pad1;
  int64_t dur, bytes, alloc, free_;
};
static_assert(sizeof(Op) == 48, "record layout");

struct Topo {
  int32_t tp, pp, dp, ep, vpp, order;
};

enum { OK = 0, E_INVALID_ARG = 1, E_INVALID_SPEC = 2, E_MISMATCH = 4, E_DEADLOCK = 5, E_NEGMEM = 6 };

struct Coords {
  int64_t tp, pp, dp, ep, edp;
};

Coords coords_of(const Topo &t, int64_t r) {
  Coords c;
  c.tp = r % t.tp;
  if (t.order == 1) {  // tp-cp-ep-dp-pp: TP fastest, then DP, then PP
    c.dp = (r / t.tp) % t.dp;
    c.pp = r / ((int64_t)t.tp * t.dp);
  } else {  // TP fastest, then PP, then DP
    c.pp = (r / t.tp) % t.pp;
    c.dp = r / ((int64_t)t.tp * t.pp);
  }
  c.ep = c.dp % t.ep;
  c.edp = c.dp / t.ep;
  return c;
}

int64_t rank_of(const Topo &t, int64_t tp_i, int64_t pp_i, int64_t dp_i) {
  if (t.order == 1) return tp_i + (int64_t)t.tp * (dp_i + (int64_t)t.dp * pp_i);
  return tp_i + (int64_t)t.tp * (pp_i + (int64_t)t.pp * dp_i);
}

// Concrete group id of a role for a rank (closed form in its coordinates).
int64_t group_id(const Topo &t, int role, const Coords &c) {
  switch (role) {
    case 1: return c.pp + (int64_t)t.pp * c.dp;                        // TP: one per (pp, dp)
    case 2: return c.tp + (int64_t)t.tp * c.pp;                        // DP: one per (tp, pp)
    case 3: return c.tp + (int64_t)t.tp * (c.pp + (int64_t)t.pp * c.edp);  // EP: per (tp, pp, edp)
    case 4: return c.tp + (int64_t)t.tp * (c.pp + (int64_t)t.pp * c.ep);   // EDP: per (tp, pp, ep)
    default: return 0;                                                 // WORLD
  }
}

int64_t role_size(const Topo &t, int role) {
  switch (role) {
    case 1: return t.tp;
    case 2: return t.dp;
    case 3: return t.ep;
    case 4: return t.dp / t.ep;
    default: return (int64_t)t.tp * t.pp * t.dp;
  }
}

uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// Reading Z8: d' = (d * (65536 + delta)) >> 16, delta = ((h >> 40) mod (2 amp + 1)) - amp.
int64_t perturb(int64_t d, uint64_t uid, int k, uint64_t seed, int amp) {
  if (k == 0 || amp == 0) return d;
  uint64_t x = seed ^ ((uint64_t)k * 0x9E3779B97F4A7C15ULL) ^ (uid * 0xBF58476D1CE4E5B9ULL);
  uint64_t h = splitmix64(x);
  int64_t delta = (int64_t)((h >> 40) % (uint64_t)(2 * amp + 1)) - amp;
  return (d * (65536 + delta)) >> 16;
}

struct Group {
  int role = 0;       // 1..5 collectives, 6 P2P message
  int coll = -1;
  uint64_t uid = 0;
  int64_t dur = 0;    // max over members' op durations (reading Z2)
  int64_t expect = 0; // expected member count
  std::vector<int32_t> members;
  int senders = 0, receivers = 0;
};

struct Graph {
  int64_t W = 0, N = 0;
  std::vector<int64_t> rank_base;  // [W+1]
  std::vector<int32_t> node_rank;
  std::vector<int32_t> node_tidx;
  std::vector<const Op *> node_op;
  std::vector<std::vector<int32_t>> node_groups;  // group indices per node (in insertion order)
  std::vector<Group> groups;
  std::vector<int64_t> static_of_rank;
  // row f2 (multi-stream ranks): the previous op issued on the node's stream, and the latest op
  // issued before it that records the event slot it waits on (-1 = none)
  std::vector<int32_t> spred, esrc;
  // rows f1/f3/f4: optional per-node overrides of the template durations / memory deltas
  const int64_t *nd_ov = nullptr, *alloc_ov = nullptr, *free_ov = nullptr;
  std::string err;
};

// Rows f1/f3/f4 (P:1170-1179 calibration, P:1767-1773 what-if, P:1745-1748 MoE imbalance): node n
// lasts node_dur[n] instead of its template duration; a synchronization group lasts the max of its
// members' durations (reading Z2, unchanged); memory deltas likewise per node.
int apply_overrides(Graph &g, const int64_t *node_dur, const int64_t *node_alloc, const int64_t *node_free) {
  g.nd_ov = node_dur;
  g.alloc_ov = node_alloc;
  g.free_ov = node_free;
  if (node_dur) {
    for (int64_t n = 0; n < g.N; ++n)
      if (node_dur[n] < 0 || node_dur[n] > (1LL << 40)) { g.err = "node duration out of range"; return E_INVALID_ARG; }
    for (auto &G : g.groups) {
      G.dur = 0;
      for (int32_t m : G.members) G.dur = std::max(G.dur, node_dur[m]);
    }
  }
  if (node_alloc || node_free)
    for (int64_t n = 0; n < g.N; ++n)
      if ((node_alloc && node_alloc[n] < 0) || (node_free && node_free[n] < 0)) { g.err = "negative memory delta"; return E_INVALID_ARG; }
  return OK;
}

int expand(const Topo &t, const Op *ops, int64_t n_ops, const int64_t *tmpl_ptr,
           const int64_t *static_mem, Graph &g) {
  if (t.tp < 1 || t.pp < 1 || t.dp < 1 || t.ep < 1 || t.dp % t.ep != 0 || (t.order != 0 && t.order != 1)) {
    g.err = "invalid topology";
    return E_INVALID_SPEC;
  }
  if (tmpl_ptr[0] != 0 || tmpl_ptr[t.pp] != n_ops) { g.err = "tmpl_ptr"; return E_INVALID_ARG; }
  for (int s = 0; s < t.pp; ++s)
    if (tmpl_ptr[s + 1] < tmpl_ptr[s]) { g.err = "tmpl_ptr not monotone"; return E_INVALID_ARG; }
  for (int64_t i = 0; i < n_ops; ++i) {
    const Op &o = ops[i];
    bool ok = o.kind <= 2 && o.stream < 4 && o.ev_record <= 8 && o.ev_wait <= 8 && o.dur >= 0 && o.dur <= (1LL << 40) && o.bytes >= 0 &&
              o.alloc >= 0 && o.free_ >= 0;
    if (o.kind == 1) ok = ok && o.role >= 1 && o.role <= 5 && o.coll <= 5;
    if (o.kind == 2) ok = ok && o.p2p_mask >= 1 && o.p2p_mask <= 15 && t.pp > 1;
    if (!ok) { g.err = "malformed op " + std::to_string(i); return E_INVALID_ARG; }
  }
  // memory never negative in program order (per template; every rank of a stage shares it)
  for (int s = 0; s < t.pp; ++s) {
    int64_t run = 0;
    for (int64_t i = tmpl_ptr[s]; i < tmpl_ptr[s + 1]; ++i) {
      run += ops[i].alloc;
      run -= ops[i].free_;
      if (run < 0) { g.err = "negative memory in stage " + std::to_string(s); return E_NEGMEM; }
    }
  }
  const int64_t W = (int64_t)t.tp * t.pp * t.dp;
  g.W = W;
  g.rank_base.assign(W + 1, 0);
  for (int64_t r = 0; r < W; ++r) {
    Coords c = coords_of(t, r);
    g.rank_base[r + 1] = g.rank_base[r] + (tmpl_ptr[c.pp + 1] - tmpl_ptr[c.pp]);
  }
  g.N = g.rank_base[W];
  g.node_rank.resize(g.N);
  g.node_tidx.resize(g.N);
  g.node_op.resize(g.N);
  g.node_groups.assign(g.N, {});
  g.spred.assign(g.N, -1);
  g.esrc.assign(g.N, -1);
  g.static_of_rank.resize(W);

  // key: (role, gid, occurrence) -> group index
  std::map<std::tuple<int, int64_t, int64_t>, int32_t> index;
  auto get_group = [&](int role, int64_t gid, int64_t occ) -> int32_t {
    auto key = std::make_tuple(role, gid, occ);
    auto it = index.find(key);
    if (it != index.end()) return it->second;
    int32_t id = (int32_t)g.groups.size();
    Group G;
    G.role = role;
    G.uid = ((uint64_t)role << 56) | ((uint64_t)gid << 24) | (uint64_t)occ;
    G.expect = role == 6 ? 2 : role_size(t, role);
    g.groups.push_back(G);
    index.emplace(key, id);
    return id;
  };

  for (int64_t r = 0; r < W; ++r) {
    Coords c = coords_of(t, r);
    int64_t s = c.pp;
    g.static_of_rank[r] = static_mem[s];
    int64_t prev_rank = rank_of(t, c.tp, (s - 1 + t.pp) % t.pp, c.dp);
    int64_t next_rank = rank_of(t, c.tp, (s + 1) % t.pp, c.dp);
    int32_t last_on[4] = {-1, -1, -1, -1}, last_rec[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
    int64_t occ_role[6] = {0, 0, 0, 0, 0, 0};
    int64_t occ_bit[4] = {0, 0, 0, 0};
    for (int64_t i = tmpl_ptr[s]; i < tmpl_ptr[s + 1]; ++i) {
      int64_t ti = i - tmpl_ptr[s];
      int32_t n = (int32_t)(g.rank_base[r] + ti);
      const Op &o = ops[i];
      g.node_rank[n] = (int32_t)r;
      g.node_tidx[n] = (int32_t)ti;
      g.node_op[n] = &o;
      g.spred[n] = last_on[o.stream];
      g.esrc[n] = o.ev_wait ? last_rec[o.ev_wait - 1] : -1;
      last_on[o.stream] = n;
      if (o.ev_record) last_rec[o.ev_record - 1] = n;
      if (o.kind == 1) {
        int64_t occ = occ_role[o.role]++;
        int32_t gi = get_group(o.role, group_id(t, o.role, c), occ);
        Group &G = g.groups[gi];
        if (G.coll < 0) G.coll = o.coll;
        else if (G.coll != o.coll) { g.err = "collective type mismatch"; return E_MISMATCH; }
        G.members.push_back(n);
        G.dur = std::max(G.dur, o.dur);
        g.node_groups[n].push_back(gi);
      } else if (o.kind == 2) {
        for (int b = 0; b < 4; ++b) {
          if (!(o.p2p_mask & (1 << b))) continue;
          int64_t occ = occ_bit[b]++;
          int64_t sender, dir;
          bool is_send;
          switch (b) {
            case 0: sender = r; dir = 0; is_send = true; break;            // SEND_NEXT
            case 1: sender = prev_rank; dir = 0; is_send = false; break;   // RECV_PREV
            case 2: sender = r; dir = 1; is_send = true; break;            // SEND_PREV
            default: sender = next_rank; dir = 1; is_send = false; break;  // RECV_NEXT
          }
          int32_t gi = get_group(6, sender * 2 + dir, occ);
          Group &G = g.groups[gi];
          G.members.push_back(n);
          G.dur = std::max(G.dur, o.dur);
          if (is_send) G.senders++; else G.receivers++;
          g.node_groups[n].push_back(gi);
        }
      }
    }
  }
  for (size_t gi = 0; gi < g.groups.size(); ++gi) {
    Group &G = g.groups[gi];
    if ((int64_t)G.members.size() != G.expect || (G.role == 6 && (G.senders != 1 || G.receivers != 1))) {
      g.err = "sync group " + std::to_string(gi) + " (role " + std::to_string(G.role) + ") has " +
              std::to_string(G.members.size()) + " of " + std::to_string(G.expect) + " members";
      return E_MISMATCH;
    }
    std::sort(G.members.begin(), G.members.end());
  }
  return OK;
}

int64_t node_duration(const Graph &g, int32_t n, int k, uint64_t seed, int amp, uint32_t mask) {
  const int64_t d = g.nd_ov ? g.nd_ov[n] : g.node_op[n]->dur;
  if (!(mask & 1u)) return d;
  uint64_t uid = ((uint64_t)g.node_rank[n] << 32) | (uint64_t)(uint32_t)g.node_tidx[n];
  return perturb(d, uid, k, seed, amp);
}

int64_t group_dur(const Group &G, int k, uint64_t seed, int amp, uint32_t mask) {
  uint32_t bit = G.role == 6 ? 4u : 2u;
  if (!(mask & bit)) return G.dur;
  return perturb(G.dur, G.uid, k, seed, amp);
}

// Discrete-event replay of one scenario. gdur[gi] and ndur(n) are the (perturbed) durations.
int replay(const Graph &g, const std::function<int64_t(int32_t)> &ndur,
           const std::vector<int64_t> &gdur, std::vector<int64_t> &start,
           std::vector<int64_t> &finish, std::string &err) {
  const int64_t N = g.N;
  start.assign(N, 0);
  finish.assign(N, 0);
  std::vector<int32_t> pend(N, 0);
  std::vector<int64_t> contrib(N, 0), gstart_max(N, 0);
  for (int64_t n = 0; n < N; ++n) pend[n] = (int32_t)g.node_groups[n].size();
  std::vector<int32_t> arrived(g.groups.size(), 0);
  std::vector<int64_t> gready(g.groups.size(), 0);
  using Ev = std::pair<int64_t, int32_t>;
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> heap;
  int64_t done = 0;

  auto release = [&](int32_t n, int64_t t) {
    if (g.node_groups[n].empty()) {  // compute span: wait out the duration
      start[n] = t;
      heap.push({t + ndur(n), n});
      return;
    }
    for (int32_t gi : g.node_groups[n]) {  // synchronization: all must reach it
      arrived[gi]++;
      gready[gi] = std::max(gready[gi], t);
      const Group &G = g.groups[gi];
      if (arrived[gi] == (int32_t)G.members.size()) {
        int64_t gs = gready[gi];
        int64_t gf = gs + gdur[gi];
        for (int32_t m : G.members) {
          contrib[m] = std::max(contrib[m], gf);
          gstart_max[m] = std::max(gstart_max[m], gs);
          if (--pend[m] == 0) {
            start[m] = gstart_max[m];
            heap.push({contrib[m], m});
          }
        }
      }
    }
  };
  // directional edges ("one operation must complete before another begins"): the stream
  // predecessor and, row f2, the event source; a node is released once all have finished
  std::vector<int32_t> deps(N, 0);
  std::vector<int64_t> rdy(N, 0);
  // successor lists as a CSR (succ_ptr / succ)
  std::vector<int64_t> succ_ptr(N + 1, 0);
  for (int64_t n = 0; n < N; ++n) {
    if (g.spred[n] >= 0) { ++deps[n]; ++succ_ptr[g.spred[n] + 1]; }
    if (g.esrc[n] >= 0) { ++deps[n]; ++succ_ptr[g.esrc[n] + 1]; }
  }
  for (int64_t n = 0; n < N; ++n) succ_ptr[n + 1] += succ_ptr[n];
  std::vector<int32_t> succ(succ_ptr[N]);
  {
    std::vector<int64_t> fill(succ_ptr.begin(), succ_ptr.end() - 1);
    for (int64_t n = 0; n < N; ++n) {
      if (g.spred[n] >= 0) succ[fill[g.spred[n]]++] = (int32_t)n;
      if (g.esrc[n] >= 0) succ[fill[g.esrc[n]]++] = (int32_t)n;
    }
  }
  for (int64_t n = 0; n < N; ++n)
    if (deps[n] == 0) release((int32_t)n, 0);
  while (!heap.empty()) {
    Ev e = heap.top();
    heap.pop();
    int32_t n = e.second;
    finish[n] = e.first;
    ++done;
    for (int64_t x = succ_ptr[n]; x < succ_ptr[n + 1]; ++x) {
      const int32_t d = succ[x];
      rdy[d] = std::max(rdy[d], e.first);
      if (--deps[d] == 0) release(d, rdy[d]);
    }
  }
  if (done != N) {
    int64_t incomplete = 0;
    for (size_t gi = 0; gi < g.groups.size(); ++gi)
      if (arrived[gi] != (int32_t)g.groups[gi].members.size()) ++incomplete;
    err = "deadlock: " + std::to_string(N - done) + " nodes never finished, " +
          std::to_string(incomplete) + " sync groups incomplete";
    return E_DEADLOCK;
  }
  return OK;
}

int peak_memory(const Graph &g, const std::vector<int64_t> &start, const std::vector<int64_t> &finish,
                int64_t *peak_out, std::string &err) {
  for (int64_t r = 0; r < g.W; ++r) {
    // (time, event index, delta): +alloc at start (index 2i), -free at finish (index 2i+1)
    std::vector<std::tuple<int64_t, int64_t, int64_t>> ev;
    for (int64_t n = g.rank_base[r]; n < g.rank_base[r + 1]; ++n) {
      int64_t i = n - g.rank_base[r];
      ev.emplace_back(start[n], 2 * i, g.alloc_ov ? g.alloc_ov[n] : g.node_op[n]->alloc);
      ev.emplace_back(finish[n], 2 * i + 1, -(g.free_ov ? g.free_ov[n] : g.node_op[n]->free_));
    }
    std::sort(ev.begin(), ev.end());
    int64_t run = 0, best = 0;
    for (auto &e : ev) {
      run += std::get<2>(e);
      if (run < 0) { err = "negative memory on rank " + std::to_string(r); return E_NEGMEM; }
      best = std::max(best, run);
    }
    peak_out[r] = g.static_of_rank[r] + best;
  }
  return OK;
}

thread_local std::string g_last;

void put_err(char *err, int errlen, const std::string &m) {
  g_last = m;
  if (err && errlen > 0) {
    std::snprintf(err, (size_t)errlen, "%s", m.c_str());
  }
}

}  // namespace

extern "C" {

// stats_out[8]: world, nodes, groups, memberships, levels, sync nodes, max group size, 0.
// level_out (optional, [n_groups]): level of each group in the oracle's group order.
// Group export (optional): grp_uid_out[G], grp_dur_out[G], grp_ptr_out[G+1], grp_mem_out[M].
int oracle_expand(const Topo *t, const Op *ops, int64_t n_ops, const int64_t *tmpl_ptr,
                  const int64_t *static_mem, int64_t *stats_out, uint64_t *grp_uid_out,
                  int64_t *grp_dur_out, int64_t *grp_ptr_out, int32_t *grp_mem_out,
                  int64_t *grp_level_out, char *err, int errlen) {
  Graph g;
  int st = expand(*t, ops, n_ops, tmpl_ptr, static_mem, g);
  if (st) { put_err(err, errlen, g.err); return st; }
  int64_t M = 0, sync_nodes = 0, maxsz = 0;
  for (auto &G : g.groups) { M += (int64_t)G.members.size(); maxsz = std::max<int64_t>(maxsz, G.members.size()); }
  for (int64_t n = 0; n < g.N; ++n) sync_nodes += !g.node_groups[n].empty();
  // Levels (reading of SURVEY §8 a5): lvl(g) = 1 + max over members n of lvl(prev-sync(n)),
  // lvl(node) = max over its groups, 0 before the first sync node. This is exactly the replay
  // with every compute span lasting 0 and every group lasting 1: the finish time of a sync node
  // is then its level (finish(prev-sync) = ready(n); group finish = max ready + 1).
  std::vector<int64_t> lv_start, lv_fin, unit(g.groups.size(), 1);
  std::string e2;
  st = replay(g, [](int32_t) { return (int64_t)0; }, unit, lv_start, lv_fin, e2);
  if (st) { put_err(err, errlen, e2); return st; }
  int64_t levels = 0;
  std::vector<int64_t> glevel(g.groups.size(), 0);
  for (size_t gi = 0; gi < g.groups.size(); ++gi) {
    int64_t mx = 0;
    for (int32_t m : g.groups[gi].members) {
      // ready(m) = finish of its directional predecessors (stream, event source), 0 if none
      int64_t ready = 0;
      if (g.spred[m] >= 0) ready = std::max(ready, lv_fin[g.spred[m]]);
      if (g.esrc[m] >= 0) ready = std::max(ready, lv_fin[g.esrc[m]]);
      mx = std::max(mx, ready);
    }
    glevel[gi] = mx + 1;
    levels = std::max(levels, glevel[gi]);
  }
  if (stats_out) {
    stats_out[0] = g.W; stats_out[1] = g.N; stats_out[2] = (int64_t)g.groups.size(); stats_out[3] = M;
    stats_out[4] = levels; stats_out[5] = sync_nodes; stats_out[6] = maxsz; stats_out[7] = 0;
  }
  if (grp_ptr_out) {
    int64_t off = 0;
    for (size_t gi = 0; gi < g.groups.size(); ++gi) {
      const Group &G = g.groups[gi];
      if (grp_uid_out) grp_uid_out[gi] = G.uid;
      if (grp_dur_out) grp_dur_out[gi] = G.dur;
      if (grp_level_out) grp_level_out[gi] = glevel[gi];
      grp_ptr_out[gi] = off;
      for (int32_t m : G.members) grp_mem_out[off++] = m;
    }
    grp_ptr_out[g.groups.size()] = off;
  }
  return OK;
}

// Replays n_scen scenarios (scenario indices k = scen_first .. scen_first+n_scen-1).
// iter_out[n_scen] (required); rank_end_out[n_scen][W], peak_out[n_scen][W],
// start_out/finish_out[n_scen][N] optional (NULL = not written). n_threads >= 1.
// Overrides (rows f1/f3/f4, optional, [N] in the oracle's node order = rank-major program order):
// node_dur replaces the template durations (groups last the max of their members'), node_alloc /
// node_free the memory deltas.
int oracle_replay_ov(const Topo *t, const Op *ops, int64_t n_ops, const int64_t *tmpl_ptr,
                     const int64_t *static_mem, const int64_t *node_dur, const int64_t *node_alloc,
                     const int64_t *node_free, int32_t scen_first, int32_t n_scen, uint64_t seed,
                     int32_t amp, uint32_t kind_mask, int64_t *iter_out, int64_t *rank_end_out,
                     int64_t *peak_out, int64_t *start_out, int64_t *finish_out, int32_t n_threads,
                     char *err, int errlen) {
  if (n_scen < 0 || amp < 0 || amp > 65535 || n_threads < 1 || !iter_out) {
    put_err(err, errlen, "bad arguments");
    return E_INVALID_ARG;
  }
  Graph g;
  int st = expand(*t, ops, n_ops, tmpl_ptr, static_mem, g);
  if (st) { put_err(err, errlen, g.err); return st; }
  st = apply_overrides(g, node_dur, node_alloc, node_free);
  if (st) { put_err(err, errlen, g.err); return st; }
  std::vector<int> status(n_scen, OK);
  std::vector<std::string> msgs(n_scen);
  auto work = [&](int tid) {
    std::vector<int64_t> start, finish, gd(g.groups.size());
    for (int j = tid; j < n_scen; j += n_threads) {
      int k = scen_first + j;
      for (size_t gi = 0; gi < g.groups.size(); ++gi) gd[gi] = group_dur(g.groups[gi], k, seed, amp, kind_mask);
      auto nd = [&](int32_t n) { return node_duration(g, n, k, seed, amp, kind_mask); };
      int s2 = replay(g, nd, gd, start, finish, msgs[j]);
      if (s2) { status[j] = s2; continue; }
      int64_t T = 0;
      for (int64_t n = 0; n < g.N; ++n) T = std::max(T, finish[n]);
      iter_out[j] = T;
      if (rank_end_out)
        for (int64_t r = 0; r < g.W; ++r)
          rank_end_out[(int64_t)j * g.W + r] = g.rank_base[r + 1] > g.rank_base[r] ? finish[g.rank_base[r + 1] - 1] : 0;
      if (peak_out) {
        int s3 = peak_memory(g, start, finish, peak_out + (int64_t)j * g.W, msgs[j]);
        if (s3) { status[j] = s3; continue; }
      }
      if (start_out) std::copy(start.begin(), start.end(), start_out + (int64_t)j * g.N);
      if (finish_out) std::copy(finish.begin(), finish.end(), finish_out + (int64_t)j * g.N);
    }
  };
  int nt = std::min<int>(n_threads, std::max(1, n_scen));
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int i = 0; i < nt; ++i) th.emplace_back(work, i);
    for (auto &x : th) x.join();
  }
  for (int j = 0; j < n_scen; ++j)
    if (status[j]) { put_err(err, errlen, msgs[j]); return status[j]; }
  return OK;
}

int oracle_replay(const Topo *t, const Op *ops, int64_t n_ops, const int64_t *tmpl_ptr,
                  const int64_t *static_mem, int32_t scen_first, int32_t n_scen, uint64_t seed,
                  int32_t amp, uint32_t kind_mask, int64_t *iter_out, int64_t *rank_end_out,
                  int64_t *peak_out, int64_t *start_out, int64_t *finish_out, int32_t n_threads,
                  char *err, int errlen) {
  return oracle_replay_ov(t, ops, n_ops, tmpl_ptr, static_mem, nullptr, nullptr, nullptr, scen_first, n_scen,
                          seed, amp, kind_mask, iter_out, rank_end_out, peak_out, start_out, finish_out,
                          n_threads, err, errlen);
}

// Row f3 (what-if attribution): the critical path of scenario k, walked back from the
// node that finishes last (T; lowest node id on ties). A compute node was started by its stream
// predecessor. A synchronization node finished with the group reaching the max (start + dur') over
// its groups (lowest uid on ties); that group started when its latest member became ready (max
// ready = finish of the member's stream predecessor; lowest member id on ties), so the walk
// continues at that member's predecessor; it stops at a node whose start is 0 with no predecessor
// edge (a node's predecessor: its stream predecessor or event source, whichever finished later,
// the lower id on ties). path_out receives the visited nodes, last first (n_out = count; capacity cap).
int oracle_critical_path(const Topo *t, const Op *ops, int64_t n_ops, const int64_t *tmpl_ptr,
                         const int64_t *static_mem, const int64_t *node_dur, int32_t k, uint64_t seed,
                         int32_t amp, uint32_t kind_mask, int32_t *path_out, int64_t cap, int64_t *n_out,
                         int64_t *T_out, char *err, int errlen) {
  Graph g;
  int st = expand(*t, ops, n_ops, tmpl_ptr, static_mem, g);
  if (st) { put_err(err, errlen, g.err); return st; }
  st = apply_overrides(g, node_dur, nullptr, nullptr);
  if (st) { put_err(err, errlen, g.err); return st; }
  std::vector<int64_t> gd(g.groups.size()), start, finish;
  for (size_t gi = 0; gi < g.groups.size(); ++gi) gd[gi] = group_dur(g.groups[gi], k, seed, amp, kind_mask);
  std::string e2;
  st = replay(g, [&](int32_t n) { return node_duration(g, n, k, seed, amp, kind_mask); }, gd, start, finish, e2);
  if (st) { put_err(err, errlen, e2); return st; }
  int64_t T = 0;
  int32_t cur = -1;
  for (int64_t n = 0; n < g.N; ++n)
    if (finish[n] > T || cur < 0) {
      if (cur < 0 || finish[n] > T) { T = finish[n]; cur = (int32_t)n; }
    }
  if (T_out) *T_out = T;
  int64_t len = 0;
  // a node's ready time is the finish of its latest directional predecessor (stream predecessor
  // or, row f2, event source; the lower node id on ties), 0 without one
  auto pred = [&](int32_t n) -> int32_t {
    const int32_t a = g.spred[n], b = g.esrc[n];
    if (a < 0) return b;
    if (b < 0) return a;
    if (finish[a] != finish[b]) return finish[a] > finish[b] ? a : b;
    return std::min(a, b);
  };
  auto ready = [&](int32_t m) { const int32_t p = pred(m); return p < 0 ? (int64_t)0 : finish[p]; };
  while (cur >= 0) {
    if (len < cap && path_out) path_out[len] = cur;
    ++len;
    int32_t next = -1;
    if (g.node_groups[cur].empty()) {
      next = pred(cur);
    } else {
      int32_t best = -1;
      int64_t bf = -1;
      for (int32_t gi : g.node_groups[cur]) {
        int64_t gs = 0;
        for (int32_t m : g.groups[gi].members) gs = std::max(gs, ready(m));
        const int64_t f = gs + gd[gi];
        if (f > bf || (f == bf && g.groups[gi].uid < g.groups[best].uid)) { bf = f; best = gi; }
      }
      const Group &G = g.groups[best];
      int32_t mstar = -1;
      int64_t mr = -1;
      for (int32_t m : G.members)  // members sorted by id: the first max is the lowest id
        if (ready(m) > mr) { mr = ready(m); mstar = m; }
      next = pred(mstar);
    }
    cur = next;
  }
  if (n_out) *n_out = len;
  return OK;
}

// Row f4, the MoE mock router (App. F): "The br represents the ratio of the actual data
// volume possessed by a specific rank to the volume it would possess under a perfectly uniform
// distribution ... multiple gating operations occur, each requiring control via br". A rank whose
// EP coordinate is e processes br[v][e] times the uniform share of gating event v's tokens, so the
// work and the buffers of every op routed by event v on that rank scale by it (reading R7):
// x' = floor(x * br / 65536) with br in Q16. Plain loops over ranks and their template ops, in the
// oracle's node order (rank-major, program order); base values = the template's unless given.
// scale bits: 1 duration, 2 allocation, 4 free.
int oracle_moe_load(const Topo *t, const Op *ops, int64_t n_ops, const int64_t *tmpl_ptr,
                    const int32_t *op_event, const int32_t *br_q16, int32_t n_events, uint32_t scale,
                    const int64_t *base_dur, const int64_t *base_alloc, const int64_t *base_free,
                    int64_t *dur_out, int64_t *alloc_out, int64_t *free_out) {
  const int64_t W = (int64_t)t->tp * t->pp * t->dp;
  int64_t n = 0;
  for (int64_t r = 0; r < W; ++r) {
    const Coords c = coords_of(*t, r);
    for (int64_t i = tmpl_ptr[c.pp]; i < tmpl_ptr[c.pp + 1]; ++i, ++n) {
      if (i >= n_ops) return E_INVALID_ARG;
      int64_t d = base_dur ? base_dur[n] : ops[i].dur;
      int64_t a = base_alloc ? base_alloc[n] : ops[i].alloc;
      int64_t f = base_free ? base_free[n] : ops[i].free_;
      const int32_t v = op_event[i];
      if (v >= n_events) return E_INVALID_ARG;
      if (v >= 0) {
        const int64_t br = br_q16[(int64_t)v * t->ep + c.ep];  // this rank's share of event v
        if (scale & 1) d = d * br / 65536;  // non-negative operands: division = floor
        if (scale & 2) a = a * br / 65536;
        if (scale & 4) f = f * br / 65536;
      }
      dur_out[n] = d;
      alloc_out[n] = a;
      free_out[n] = f;
    }
  }
  return OK;
}

uint64_t oracle_splitmix64(uint64_t x) { return splitmix64(x); }
int64_t oracle_perturb(int64_t d, uint64_t uid, int32_t k, uint64_t seed, int32_t amp) {
  return perturb(d, uid, k, seed, amp);
}

}  // extern "C"
