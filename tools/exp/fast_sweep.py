"""Dev experiment: C5 (or $CFG) replay time under PRISM_POLL_FAST / PRISM_POLL policies, one subprocess each."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import sys; sys.path.insert(0, %r)
import torch
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config(%r)
g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
ts = []
for _ in range(6):
    it = g.replay(64, amp_q16=6554, kind_mask=7, algo="cells")
    ts.append(g.last_timing()["levels"])
print("RESULT", min(ts), sorted(ts)[3], int(it.sum() %% (1 << 61)))
'''
cfg = os.environ.get("CFG", "C5")
for pol in sys.argv[1:]:
    fast, _, slow = pol.partition("/")
    env = dict(os.environ, PRISM_POLL_FAST=fast)
    if slow: env["PRISM_POLL"] = slow
    r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg)], env=env, capture_output=True, text=True)
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
    print(cfg, pol, line[0] if line else r.stderr[-500:], flush=True)
