// plan.cpp — host-side validation and quotient analysis for prism_build_graph.
//
// Everything here is O(template ops), independent of the world size: the per-stage templates are
// shared by all tp*dp ranks of a stage (§5.2 "execution graphs are identical across DP
// groups"), so every concrete synchronization group is an instance of a *quotient group* — one
// template-level collective occurrence or P2P message — and all instances of a quotient group
// have the same member template positions, the same duration and the same frontier level. The
// per-node / per-membership work (rows a3, a4) runs on the GPU in expand.cu.
//
// Group semantics (§5.1; readings Z1-Z3, Z10 in DESIGN.md §3):
//   * the k-th collective of role R in template s forms, for every concrete R group of stage s,
//     the k-th occurrence of that group (all members run template s, so all members sit at the
//     same template index); WORLD collectives pair the k-th WORLD op of every stage;
//   * the k-th SEND_NEXT of stage s pairs with the k-th RECV_PREV of stage (s+1) mod pp, the k-th
//     SEND_PREV of stage s with the k-th RECV_NEXT of stage (s-1) mod pp (same tp/dp coords).
// Levels (row a5): lvl(g) = 1 + max over members n of lvl(prev-sync(n)), lvl(node) = max over its
// groups; computed on the quotient graph by a structural replay with per-stage cursors. A stage
// whose cursor cannot advance past a sync op means a cyclic synchronization structure:
// PRISM_E_DEADLOCK.
#include <algorithm>
#include <cstdio>
#include <numeric>
#include <string>
#include <vector>

#include "prism_internal.h"

#ifdef PLAN_TIMING
#include <chrono>
#define TMARK(name) do { auto _n = std::chrono::high_resolution_clock::now(); \
  std::fprintf(stderr, "  %-12s %.3f ms\n", name, std::chrono::duration<double, std::milli>(_n - _t).count()); _t = _n; } while (0)
#else
#define TMARK(name)
#endif

namespace prism {

namespace {

int64_t role_size(const Topo &t, int role) {
  switch (role) {
    case PRISM_ROLE_TP: return t.tp;
    case PRISM_ROLE_DP: return t.dp;
    case PRISM_ROLE_EP: return t.ep;
    case PRISM_ROLE_EDP: return t.dp / t.ep;
    default: return (int64_t)t.tp * t.pp * t.dp;
  }
}

std::string fmt(const char *f, long long a = 0, long long b = 0, long long c = 0) {
  char buf[256];
  std::snprintf(buf, sizeof buf, f, a, b, c);
  return buf;
}

}  // namespace

prism_status plan_graph(const prism_topology &tp_, const prism_templates &tm, Plan &P,
                        std::string &err) {
  Topo t{tp_.tp, tp_.pp, tp_.dp, tp_.ep, tp_.rank_order};
  if (t.tp < 1 || t.pp < 1 || t.dp < 1 || t.ep < 1 || t.dp % t.ep != 0 ||
      (t.order != PRISM_ORDER_TP_PP_DP && t.order != PRISM_ORDER_MEGATRON)) {
    err = fmt("invalid topology tp=%lld pp=%lld dp=%lld", t.tp, t.pp, t.dp) +
          fmt(" ep=%lld order=%lld", t.ep, t.order);
    return PRISM_E_INVALID_SPEC;
  }
  const int64_t W = (int64_t)t.tp * t.pp * t.dp;
  if (W > (1LL << 30)) { err = "world too large"; return PRISM_E_INVALID_SPEC; }
  if (tm.n_ops < 0 || (tm.n_ops > 0 && !tm.ops) || !tm.tmpl_ptr || !tm.static_mem) {
    err = "null template arrays";
    return PRISM_E_INVALID_ARG;
  }
  if (tm.tmpl_ptr[0] != 0 || tm.tmpl_ptr[t.pp] != tm.n_ops) {
    err = "tmpl_ptr must start at 0 and end at n_ops";
    return PRISM_E_INVALID_ARG;
  }
#ifdef PLAN_TIMING
  auto _t = std::chrono::high_resolution_clock::now();
#endif
  P = Plan();
  P.topo = t;
  P.W = W;
  const int pp = t.pp;
  P.stage_len.resize(pp);
  P.stage_slots.resize(pp);
  P.stage_op0.resize(pp);
  P.t_prev_sync.assign(tm.n_ops, -1);
  P.t_slot_ptr.assign(tm.n_ops, 0);
  P.t_slots.assign(tm.n_ops, 0);

  // per stage: tidx lists of the k-th op of each role / P2P bit, and the slot of that bit
  std::vector<std::vector<int32_t>> role_ops(pp * 6), bit_ops(pp * 4), bit_slot(pp * 4);
  for (int s = 0; s < pp; ++s) {
    int64_t a = tm.tmpl_ptr[s], b = tm.tmpl_ptr[s + 1];
    if (b < a) { err = fmt("tmpl_ptr not monotone at stage %lld", s); return PRISM_E_INVALID_ARG; }
    if (b - a >= (1LL << 31)) { err = "template too long"; return PRISM_E_INVALID_ARG; }
    P.stage_len[s] = b - a;
    P.stage_op0[s] = a;
    int32_t prev = -1;
    int32_t slots = 0;
    int64_t run = 0;
    for (int64_t i = a; i < b; ++i) {
      const prism_op &o = tm.ops[i];
      int32_t ti = (int32_t)(i - a);
      bool ok = o.kind <= PRISM_KIND_P2P && o.stream < kMaxStreams && o.ev_record <= kMaxEvents &&
                o.ev_wait <= kMaxEvents && o.dur_ns >= 0 &&
                o.dur_ns <= (1LL << 40) && o.bytes >= 0 && o.mem_alloc >= 0 && o.mem_free >= 0;
      if (o.kind == PRISM_KIND_COLLECTIVE)
        ok = ok && o.role >= PRISM_ROLE_TP && o.role <= PRISM_ROLE_WORLD && o.coll <= PRISM_COLL_BARRIER;
      if (o.kind == PRISM_KIND_P2P) ok = ok && o.p2p_mask >= 1 && o.p2p_mask <= 15 && pp > 1;
      if (!ok) {
        err = fmt("malformed op %lld (stage %lld, index %lld)", i, s, ti);
        return PRISM_E_INVALID_ARG;
      }
      if (o.stream != 0 || o.ev_record || o.ev_wait) P.multistream = true;
      run += o.mem_alloc;
      run -= o.mem_free;
      if (run < 0) {
        err = fmt("running allocation of stage %lld drops below zero at template index %lld", s, ti);
        return PRISM_E_NEGATIVE_MEMORY;
      }
      P.t_prev_sync[i] = prev;
      P.t_slot_ptr[i] = slots;
      int32_t ns = 0;
      if (o.kind == PRISM_KIND_COLLECTIVE) {
        role_ops[s * 6 + o.role].push_back(ti);
        ns = 1;
      } else if (o.kind == PRISM_KIND_P2P) {
        for (int bit = 0; bit < 4; ++bit)
          if (o.p2p_mask & (1 << bit)) {
            bit_ops[s * 4 + bit].push_back(ti);
            bit_slot[s * 4 + bit].push_back(ns);
            ++ns;
          }
      }
      P.t_slots[i] = ns;
      slots += ns;
      if (ns) prev = ti;
    }
    P.stage_slots[s] = slots;
  }

  // row f2: per template op, the previous op of its stream and the event source (template
  // indices, -1 = none) and the packed stream/event byte of the cell kernel
  P.t_spred.assign(tm.n_ops, -1);
  P.t_esrc.assign(tm.n_ops, -1);
  P.t_ms.assign(tm.n_ops, 0);
  if (P.multistream) {
    // streams used, event slots renumbered densely in order of first use (the cell kernel keeps
    // (streams + events) x tp x 32 ready times per warp in shared memory)
    int8_t emap[kMaxEvents];
    for (auto &x : emap) x = -1;
    for (int64_t i = 0; i < tm.n_ops; ++i) {
      const prism_op &o = tm.ops[i];
      P.ms_streams = std::max<int32_t>(P.ms_streams, o.stream + 1);
      for (int e : {(int)o.ev_record, (int)o.ev_wait})
        if (e && emap[e - 1] < 0) emap[e - 1] = (int8_t)P.ms_events++;
    }
    for (int s = 0; s < pp; ++s) {
      int32_t last_on[kMaxStreams], last_rec[kMaxEvents];
      for (auto &x : last_on) x = -1;
      for (auto &x : last_rec) x = -1;
      for (int64_t i = tm.tmpl_ptr[s]; i < tm.tmpl_ptr[s + 1]; ++i) {
        const prism_op &o = tm.ops[i];
        const int32_t ti = (int32_t)(i - tm.tmpl_ptr[s]);
        P.t_spred[i] = last_on[o.stream];
        P.t_esrc[i] = o.ev_wait ? last_rec[o.ev_wait - 1] : -1;
        const int rec = o.ev_record ? emap[o.ev_record - 1] + 1 : 0, wt = o.ev_wait ? emap[o.ev_wait - 1] + 1 : 0;
        P.t_ms[i] = (uint16_t)(o.stream | (rec << 4) | (wt << 8));
        last_on[o.stream] = ti;
        if (o.ev_record) last_rec[o.ev_record - 1] = ti;
      }
    }
  }
  // replay classes (cell kernel) and per-stage cross-op lists
  P.t_cls.assign(tm.n_ops, 0);
  {
    // WORLD op k chains only if, on every stage, the op right before it is WORLD op k-1
    std::vector<int32_t> wk(pp, 0);
    std::vector<uint8_t> wchain;
    for (int s = 0; s < pp; ++s) {
      const int64_t a = tm.tmpl_ptr[s], b = tm.tmpl_ptr[s + 1];
      int32_t k = 0;
      for (int64_t i = a; i < b; ++i) {
        const prism_op &o = tm.ops[i];
        if (o.kind == PRISM_KIND_COLLECTIVE && o.role == PRISM_ROLE_WORLD) {
          const bool prev_world = i > a && tm.ops[i - 1].kind == PRISM_KIND_COLLECTIVE &&
                                  tm.ops[i - 1].role == PRISM_ROLE_WORLD;
          if ((int32_t)wchain.size() <= k) wchain.push_back(1);
          wchain[k] &= prev_world ? 1 : 0;
          ++k;
        }
      }
    }
    P.x_ptr.assign(pp + 1, 0);
    for (int s = 0; s < pp; ++s) {
      const int64_t a = tm.tmpl_ptr[s], b = tm.tmpl_ptr[s + 1];
      int32_t k = 0;
      for (int64_t i = a; i < b; ++i) {
        const prism_op &o = tm.ops[i];
        uint8_t c = 0;
        if (o.kind == PRISM_KIND_COLLECTIVE) {
          // the chained-collective shortcut needs a single stream (row f2)
          if (o.role == PRISM_ROLE_TP) {
            c = 1;
          } else if (o.role == PRISM_ROLE_WORLD) {
            c = (!P.multistream && k < (int32_t)wchain.size() && wchain[k]) ? 3 : 2;
            ++k;
          } else {
            const bool same = i > a && tm.ops[i - 1].kind == PRISM_KIND_COLLECTIVE && tm.ops[i - 1].role == o.role;
            c = (same && !P.multistream) ? 3 : 2;
          }
        } else if (o.kind == PRISM_KIND_P2P) {
          c = 2;
        }
        P.t_cls[i] = c;
        if (c == 2) P.x_ops.push_back(XOp{(int32_t)(i - a), P.t_slot_ptr[i], P.t_slots[i], 0});
      }
      P.x_ptr[s + 1] = (int32_t)P.x_ops.size();
      // flag 0x10: a compute span directly followed by a TP collective (the cell kernel runs the
      // pair in one iteration); consumers compare the class as t_cls & 0xF
      if (!P.multistream)
        for (int64_t i = a; i + 1 < b; ++i)
          if (P.t_cls[i] == 0 && tm.ops[i].kind == PRISM_KIND_COMPUTE && P.t_cls[i + 1] == 1) P.t_cls[i] |= 0x10;
    }
  }
  TMARK("scan");
  // ---- quotient groups --------------------------------------------------------------------
  std::vector<QGroup> Q;
  {
    size_t est = 0;
    for (auto &v : role_ops) est += v.size();
    for (auto &v : bit_ops) est += v.size();
    Q.reserve(est);
  }
  auto base_q = [](int type) {
    QGroup g{};
    g.type = type;
    g.stage2 = g.tidx2 = g.slot2 = -1;
    g.wpos = -1;
    return g;
  };
  for (int s = 0; s < pp; ++s) {
    for (int role = PRISM_ROLE_TP; role <= PRISM_ROLE_EDP; ++role) {
      const auto &L = role_ops[s * 6 + role];
      for (size_t k = 0; k < L.size(); ++k) {
        QGroup g = base_q(role);
        g.stage = s;
        g.tidx = L[k];
        g.slot = 0;
        g.size = (int32_t)role_size(t, role);
        g.inst = (int32_t)((int64_t)t.tp * t.dp / g.size);
        g.occ = (int32_t)k;
        g.dur = tm.ops[tm.tmpl_ptr[s] + L[k]].dur_ns;
        Q.push_back(g);
      }
    }
  }
  TMARK("q-coll");
  {  // WORLD: the k-th WORLD op of every stage
    size_t K = role_ops[0 * 6 + PRISM_ROLE_WORLD].size();
    for (int s = 1; s < pp; ++s)
      if (role_ops[s * 6 + PRISM_ROLE_WORLD].size() != K) {
        err = fmt("stage 0 has %lld WORLD collectives but stage %lld has %lld", (long long)K, s,
                  (long long)role_ops[s * 6 + PRISM_ROLE_WORLD].size());
        return PRISM_E_TEMPLATE_MISMATCH;
      }
    for (size_t k = 0; k < K; ++k) {
      QGroup g = base_q(PRISM_ROLE_WORLD);
      g.stage = -1;
      g.tidx = -1;
      g.slot = 0;
      g.size = (int32_t)W;
      g.inst = 1;
      g.occ = (int32_t)k;
      g.wpos = (int32_t)P.wpos.size();
      int coll = -1;
      for (int s = 0; s < pp; ++s) {
        int32_t ti = role_ops[s * 6 + PRISM_ROLE_WORLD][k];
        const prism_op &o = tm.ops[tm.tmpl_ptr[s] + ti];
        if (coll >= 0 && o.coll != coll) {
          err = fmt("WORLD collective %lld has different collective types on stages 0 and %lld", (long long)k, s);
          return PRISM_E_TEMPLATE_MISMATCH;
        }
        coll = o.coll;
        g.dur = std::max<int64_t>(g.dur, o.dur_ns);
        P.wpos.push_back(ti);
      }
      Q.push_back(g);
    }
  }
  TMARK("q-world");
  // intra-stage collective types agree trivially (one template op per quotient group)
  for (int s = 0; s < pp && pp > 1; ++s) {
    for (int dir = 0; dir < 2; ++dir) {
      int sbit = dir == 0 ? 0 : 2, rbit = dir == 0 ? 1 : 3;
      int s2 = dir == 0 ? (s + 1) % pp : (s - 1 + pp) % pp;
      const auto &S = bit_ops[s * 4 + sbit];
      const auto &R = bit_ops[s2 * 4 + rbit];
      if (S.size() != R.size()) {
        err = fmt(dir == 0 ? "stage %lld sends %lld messages to the next stage, which receives %lld"
                           : "stage %lld sends %lld messages to the previous stage, which receives %lld",
                  s, (long long)S.size(), (long long)R.size());
        return PRISM_E_TEMPLATE_MISMATCH;
      }
      for (size_t k = 0; k < S.size(); ++k) {
        QGroup g = base_q(PRISM_ROLE_P2P);
        g.stage = s;
        g.tidx = S[k];
        g.slot = bit_slot[s * 4 + sbit][k];
        g.stage2 = s2;
        g.tidx2 = R[k];
        g.slot2 = bit_slot[s2 * 4 + rbit][k];
        g.size = 2;
        g.inst = t.tp * t.dp;
        g.occ = (int32_t)k;
        g.dir = dir;
        g.dur = std::max(tm.ops[tm.tmpl_ptr[s] + S[k]].dur_ns, tm.ops[tm.tmpl_ptr[s2] + R[k]].dur_ns);
        Q.push_back(g);
      }
    }
  }
  for (auto &g : Q)
    if (g.occ >= (1 << 24)) { err = "more than 2^24 occurrences of one group"; return PRISM_E_INVALID_ARG; }

  TMARK("quotient");
  // ---- levels: structural replay on the quotient graph ------------------------------------
  // positions = (stage, template index) of sync ops; pos_q lists the quotient groups of each.
  std::vector<int64_t> pos_base(pp + 1, 0);
  for (int s = 0; s < pp; ++s) pos_base[s + 1] = pos_base[s] + P.stage_len[s];
  // pos_q: quotient groups of each position, as a CSR (positions x <= 4 groups)
  const int64_t npos_all = pos_base[pp];
  std::vector<int32_t> pq_ptr(npos_all + 1, 0), npos(Q.size());
  auto for_positions = [&](size_t qi, auto &&fn) {
    const QGroup &g = Q[qi];
    if (g.type == PRISM_ROLE_WORLD) {
      for (int s = 0; s < pp; ++s) fn(pos_base[s] + P.wpos[g.wpos + s]);
    } else if (g.type == PRISM_ROLE_P2P) {
      fn(pos_base[g.stage] + g.tidx);
      fn(pos_base[g.stage2] + g.tidx2);
    } else {
      fn(pos_base[g.stage] + g.tidx);
    }
  };
  for (size_t qi = 0; qi < Q.size(); ++qi) {
    int32_t c = 0;
    for_positions(qi, [&](int64_t x) { ++pq_ptr[x + 1]; ++c; });
    npos[qi] = c;
  }
  for (int64_t x = 0; x < npos_all; ++x) pq_ptr[x + 1] += pq_ptr[x];
  std::vector<int32_t> pq(pq_ptr[npos_all]);
  {
    std::vector<int32_t> fill(pq_ptr.begin(), pq_ptr.end() - 1);
    for (size_t qi = 0; qi < Q.size(); ++qi) for_positions(qi, [&](int64_t x) { pq[fill[x]++] = (int32_t)qi; });
  }
  std::vector<int32_t> arrived(Q.size(), 0), qlvl(Q.size(), 0), rdy(Q.size(), 0);
  std::vector<int32_t> pend(npos_all, 0), poslvl(npos_all, 0);
  for (int64_t i = 0; i < npos_all; ++i) pend[i] = pq_ptr[i + 1] - pq_ptr[i];
  std::vector<int64_t> cursor(pp, 0);
  std::vector<int32_t> curlvl(pp, 0);
  std::vector<int> work;
  auto next_sync = [&](int s, int64_t from) {
    while (from < P.stage_len[s] && pq_ptr[pos_base[s] + from + 1] == pq_ptr[pos_base[s] + from]) ++from;
    return from;
  };
  for (int s = 0; s < pp; ++s) {
    cursor[s] = next_sync(s, 0);
    work.push_back(s);
  }
  while (!work.empty()) {
    int s = work.back();
    work.pop_back();
    if (cursor[s] >= P.stage_len[s]) continue;
    const int64_t pos = pos_base[s] + cursor[s];
    for (int32_t e = pq_ptr[pos]; e < pq_ptr[pos + 1]; ++e) {
      const int32_t qi = pq[e];
      rdy[qi] = std::max(rdy[qi], curlvl[s]);
      if (++arrived[qi] == npos[qi]) {
        qlvl[qi] = rdy[qi] + 1;
        const QGroup &g = Q[qi];
        auto resolve = [&](int s2, int64_t ti) {
          int64_t p2 = pos_base[s2] + ti;
          poslvl[p2] = std::max(poslvl[p2], qlvl[qi]);
          if (--pend[p2] == 0) {
            curlvl[s2] = poslvl[p2];
            cursor[s2] = next_sync(s2, ti + 1);
            work.push_back(s2);
          }
        };
        if (g.type == PRISM_ROLE_WORLD) {
          for (int s2 = 0; s2 < pp; ++s2) resolve(s2, P.wpos[g.wpos + s2]);
        } else if (g.type == PRISM_ROLE_P2P) {
          resolve(g.stage, g.tidx);
          resolve(g.stage2, g.tidx2);
        } else {
          resolve(g.stage, g.tidx);
        }
      }
    }
  }
  for (int s = 0; s < pp; ++s)
    if (cursor[s] < P.stage_len[s]) {
      err = fmt("deadlock: stage %lld can never pass its sync op at template index %lld", s, cursor[s]);
      return PRISM_E_DEADLOCK;
    }
  for (size_t qi = 0; qi < Q.size(); ++qi) Q[qi].level = qlvl[qi];

  TMARK("levels");
  // ---- order by level, assign concrete group ids / membership ranges ----------------------
  std::vector<int32_t> ord(Q.size());
  {  // stable counting sort by level
    int32_t maxl = 0;
    for (auto &g : Q) maxl = std::max(maxl, g.level);
    std::vector<int32_t> cnt(maxl + 2, 0);
    for (auto &g : Q) ++cnt[g.level + 1];
    for (int32_t l = 0; l <= maxl; ++l) cnt[l + 1] += cnt[l];
    for (size_t qi = 0; qi < Q.size(); ++qi) ord[cnt[Q[qi].level]++] = (int32_t)qi;
  }
  P.q.resize(Q.size());
  std::vector<int32_t> new_index(Q.size());
  for (size_t i = 0; i < ord.size(); ++i) new_index[ord[i]] = (int32_t)i;
  int64_t G = 0, M = 0, X = 0, LG = 0;
  int32_t levels = 0, maxg = 0;
  for (size_t i = 0; i < ord.size(); ++i) {
    QGroup g = Q[ord[i]];
    g.gbase = G;
    g.mbase = M;
    // replay v2 cells are TP groups: a TP collective is resolved inside its cell's CTA; every
    // other group exchanges ready times through global ready slots
    g.xbase = -1;
    g.lbase = -1;
    g.cxbase = -1;
    g.clbase = -1;
    if (g.type != PRISM_ROLE_TP) {
      if (g.size <= kSmallGroup) {
        g.xbase = X;
        X += (int64_t)g.inst * g.size;
      } else {
        g.lbase = LG;
        LG += g.inst;
      }
    }
    G += g.inst;
    M += (int64_t)g.inst * g.size;
    levels = std::max(levels, g.level);
    maxg = std::max(maxg, g.size);
    P.q[i] = g;
  }
  TMARK("order");
  // per template slot tables (node-side expansion) and group-side chunks
  P.stage_slot0.assign(pp + 1, 0);
  for (int s = 0; s < pp; ++s) P.stage_slot0[s + 1] = P.stage_slot0[s] + P.stage_slots[s];
  const int64_t nslots = P.stage_slot0[pp];
  P.slot_q.assign(nslots, -1);
  P.slot_tidx.assign(nslots, 0);
  P.slot_role.assign(nslots, 0);
  P.slot_first.assign(nslots, 0);
  for (int s = 0; s < pp; ++s)
    for (int64_t i = 0; i < P.stage_len[s]; ++i) {
      const int64_t op = P.stage_op0[s] + i;
      for (int32_t u = 0; u < P.t_slots[op]; ++u) {
        const int64_t x = P.stage_slot0[s] + P.t_slot_ptr[op] + u;
        P.slot_tidx[x] = (int32_t)i;
        P.slot_first[x] = u == 0;
      }
    }
  auto put = [&](int s, int32_t tidx, int32_t slot, int32_t qnew, uint8_t role) {
    const int64_t op = P.stage_op0[s] + tidx;
    const int64_t x = P.stage_slot0[s] + P.t_slot_ptr[op] + slot;
    P.slot_q[x] = qnew;
    P.slot_role[x] = role;
  };
  for (size_t qi = 0; qi < Q.size(); ++qi) {
    const QGroup &g = Q[qi];
    const int32_t qn = new_index[qi];
    if (g.type == PRISM_ROLE_WORLD) {
      for (int s = 0; s < pp; ++s) put(s, P.wpos[g.wpos + s], 0, qn, 0);
    } else if (g.type == PRISM_ROLE_P2P) {
      put(g.stage, g.tidx, g.slot, qn, 0);
      put(g.stage2, g.tidx2, g.slot2, qn, 1);
    } else {
      put(g.stage, g.tidx, 0, qn, 0);
    }
  }
  for (int64_t x = 0; x < nslots; ++x)
    if (P.slot_q[x] < 0) { err = "internal: template slot without a group"; return PRISM_E_INVALID_ARG; }
  for (size_t i = 0; i < P.q.size(); ++i) {
    const int64_t mq = (int64_t)P.q[i].inst * P.q[i].size;
    for (int64_t off = 0; off < mq; off += 2048) {
      P.chunk_q.push_back((int32_t)i);
      P.chunk_m.push_back(off);
    }
  }
  P.t_q0.assign(tm.n_ops, -1);
  for (int s = 0; s < pp; ++s)
    for (int64_t i = 0; i < P.stage_len[s]; ++i) {
      const int64_t op = P.stage_op0[s] + i;
      if (P.t_slots[op] > 0) P.t_q0[op] = P.slot_q[P.stage_slot0[s] + P.t_slot_ptr[op]];
    }
  TMARK("slots");
  P.level_q_ptr.assign(levels + 2, 0);
  for (const auto &g : P.q) P.level_q_ptr[g.level + 1]++;
  for (int l = 0; l <= levels; ++l) P.level_q_ptr[l + 1] += P.level_q_ptr[l];
  P.levels = levels;
  P.max_group = maxg;
  P.G = G;
  P.M = M;
  P.M_cross = X;
  P.G_large = LG;
  int64_t N = 0, sync_nodes = 0;
  for (int s = 0; s < pp; ++s) {
    N += P.stage_len[s] * t.tp * t.dp;
    int64_t sn = 0;
    for (int64_t i = 0; i < P.stage_len[s]; ++i) sn += P.t_slots[P.stage_op0[s] + i] > 0;
    sync_nodes += sn * t.tp * t.dp;
  }
  P.N = N;
  P.sync_nodes = sync_nodes;
  if (N >= (1LL << 31) - 1 || M >= (1LL << 31) - 1 || G >= (1LL << 31) - 1) {
    err = fmt("graph too large for int32 ids: N=%lld M=%lld G=%lld", N, M, G);
    return PRISM_E_INVALID_ARG;
  }
  return PRISM_OK;
}

bool replica_cells_ok(const Topo &t, int32_t R) {
  return R > 1 && t.tp == 1 && t.dp % R == 0 && (t.ep == 1 || t.ep % R == 0);
}

prism_status plan_replica_cells(Plan &P, int32_t R, int32_t ks, std::string &err) {
  const Topo &t = P.topo;
  if (!replica_cells_ok(t, R)) {
    err = "replica cells need tp == 1, R | dp and (ep == 1 or R | ep)";
    return PRISM_E_INVALID_ARG;
  }
  // does a group of this role hold all R replicas of a cell (else exactly one of them)?
  auto full = [&](int role) {
    switch (role) {
      case PRISM_ROLE_DP:
      case PRISM_ROLE_WORLD: return true;
      case PRISM_ROLE_EP: return t.ep > 1;        // R | ep: the cell's replicas share edp
      case PRISM_ROLE_EDP: return t.ep == 1;      // ep = 1: the EDP group is the DP group
      default: return false;                      // TP / size-1 EP / P2P
    }
  };
  const int pp = t.pp;
  // classes: TP collectives (size-1 groups) become per-replica chained ops (flag 0x20: uid step
  // pp << 24 between replicas, gid = s + pp * dp); chained collectives of full groups keep one uid
  // for the whole cell (flag 0x40: step 0); the (compute, TP) pair flag disappears with class 1
  P.x_ops.clear();
  P.x_ptr.assign(pp + 1, 0);
  P.crec_ptr.assign(pp + 1, 0);
  for (int s = 0; s < pp; ++s) {
    const int64_t a = P.stage_op0[s], b = a + P.stage_len[s];
    for (int64_t i = a; i < b; ++i) {
      uint8_t c = P.t_cls[i] & 0xF;
      const int32_t q0 = P.t_q0[i];
      const int role = q0 >= 0 ? P.q[q0].type : 0;
      if (c == 1) c = 3 | 0x20;
      else if (c == 3) c = 3 | (full(role) ? 0x40 : 0x20);
      else if (c == 2 && ks > 1 && role == PRISM_ROLE_EP && t.ep == R * ks) c = 4;  // the CTA is the group
      P.t_cls[i] = c;
      if (c == 2)
        P.x_ops.push_back(XOp{(int32_t)(i - a), P.t_slot_ptr[i], P.t_slots[i],
                              (role != PRISM_ROLE_P2P && full(role)) ? 1 : 0});
    }
    P.x_ptr[s + 1] = (int32_t)P.x_ops.size();
    P.crec_ptr[s + 1] = P.crec_ptr[s] + (int64_t)(t.dp / R) * (P.x_ptr[s + 1] - P.x_ptr[s]);
  }
  // cell-level slots of the full groups, after the rank-level ones (the rank kernel and the level
  // path keep using those)
  int64_t X = P.M_cross, LG = P.G_large;
  for (QGroup &g : P.q) {
    if (g.type == PRISM_ROLE_P2P || !full(g.type)) continue;
    const int64_t cz = g.size / R;
    if (cz <= kSmallGroup) {
      g.cxbase = X;
      X += (int64_t)g.inst * cz;
    } else {
      g.clbase = LG;
      LG += g.inst;
    }
  }
  P.M_cross = X;
  P.G_large = LG;
  P.cell_R = R;
  P.cta_ks = ks;
  return PRISM_OK;
}

}  // namespace prism
