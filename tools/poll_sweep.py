"""Dev tool: C5 replay time under poll/backoff policies (PRISM_POLL, one subprocess each)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys; sys.path.insert(0, %r)
import torch, numpy as np
import paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
tm = w.config(%r)
g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
ts = []
for _ in range(5):
    it = g.replay(64, amp_q16=6554, kind_mask=7, algo="cells")
    ts.append(g.last_timing()["levels"])
print("RESULT", min(ts), sorted(ts)[2], int(it.sum() %% (1 << 61)))
'''


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
    pols = sys.argv[2:] or ["0,32,256", "6,32,256", "2,32,1024", "2,64,2048", "0,64,4096", "1,128,8192",
                            "4,16,512", "2,32,512"]
    ref = None
    for p in pols:  # "a,b,c" = PRISM_POLL, "F:a,b,c" = PRISM_POLL_FAST, "a,b,c+F:d,e,f" = both
        env = dict(os.environ)
        for part in p.split("+"):
            if part.startswith("F:"):
                env["PRISM_POLL_FAST"] = part[2:]
            else:
                env["PRISM_POLL"] = part
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg)], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
        if not line:
            print(p, "FAILED", r.stderr[-500:], flush=True)
            continue
        _, best, med, h = line[0].split()
        ref = ref or h
        print(f"{cfg} poll={p:28s} best={float(best):7.3f} ms med={float(med):7.3f} ms same={h == ref}", flush=True)


if __name__ == "__main__":
    main()
