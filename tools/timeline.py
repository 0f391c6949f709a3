"""Dev tool (stats build): timeline of the cross ops of one C5 pipeline (dp 0, chunk 0):
per cross op enter / deposited / detected / exit, and the handoff latency = detection - the
latest deposit among the op and its P2P partners."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
c5 = w.config("C5"); t = c5.topo
dp = int(os.environ.get("DP", "1"))
tm = w.Templates(w.Topology(t.tp, t.pp, dp, 1, t.vpp, t.rank_order), c5.ops, c5.tmpl_ptr, c5.static_mem)
g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
L = prism.lib()
amp = int(os.environ.get("AMP", "0")); rec = os.environ.get("REC", "0") == "1"
buf = (ctypes.c_ulonglong * (16 * 128 * 4))()
for _ in range(3):
    g.replay(32, amp_q16=amp, kind_mask=7, record=rec)
L.prism_debug_timeline(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(16, 128, 4).astype(np.int64)
t0 = a[a > 0].min()
print("kernel ms", g.last_timing()["levels"])
pp = t.pp
st = [tm.stage(s) for s in range(pp)]
def xlist(T):
    out = []
    for i in range(len(T)):
        o = T[i]
        if o["kind"] == 2:
            out.append(i)
        elif o["kind"] == 1 and o["role"] != 1 and not (i > 0 and T[i-1]["kind"] == 1 and T[i-1]["role"] == o["role"]):
            out.append(i)
    return out
X = [xlist(T) for T in st]
pos = [{ti: j for j, ti in enumerate(x)} for x in X]
bits = {(s, b): [i for i in range(len(st[s])) if st[s][i]["kind"] == 2 and (st[s][i]["p2p_mask"] >> b) & 1] for s in range(pp) for b in range(4)}
partners = {}
for s in range(pp):
    for sb, rb, s2 in ((0, 1, (s + 1) % pp), (2, 3, (s - 1) % pp)):
        for x, y in zip(bits[(s, sb)], bits[(s2, rb)]):
            partners.setdefault((s, x), []).append((s2, y)); partners.setdefault((s2, y), []).append((s, x))
hand, waitp, work, dep_cost, exit_cost = [], [], [], [], []
for s in range(pp):
    prev_exit = None
    for j, ti in enumerate(X[s][:128]):
        e, d, det, x = a[s, j]
        if e == 0:
            continue
        dep_cost.append(d - e); exit_cost.append(x - det)
        if prev_exit: work.append(e - prev_exit)
        prev_exit = x
        ps = partners.get((s, ti), [])
        deps = [d]
        for s2, y in ps:
            jj = pos[s2].get(y)
            if jj is not None and jj < 128 and a[s2, jj, 1] > 0:
                deps.append(a[s2, jj, 1])
        if len(deps) > 1:
            last = max(deps)
            hand.append(det - last)
            waitp.append(last - d)
def q(v):
    v = np.array(v) / 1e3
    return f"mean {v.mean():6.2f} us  p10 {np.percentile(v,10):6.2f}  p50 {np.percentile(v,50):6.2f}  p90 {np.percentile(v,90):6.2f}  (n={len(v)})"
print("deposit cost (enter->deposited)  ", q(dep_cost))
print("handoff (latest deposit->detect) ", q(hand))
print("waiting for partner             ", q(waitp))
print("exit cost (detect->exit)        ", q(exit_cost))
print("work between cross ops          ", q(work))
