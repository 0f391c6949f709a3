"""Dev tool: build one BASELINE config and run a few replays (for ncu / compute-sanitizer).

  python tools/prof_replay.py [--config C5] [--scenarios 64] [--algo cells] [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scaled", action="store_true")
    ap.add_argument("--scenarios", type=int, default=64)
    ap.add_argument("--algo", default="cells")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--record", type=int, default=1)
    args = ap.parse_args()
    import torch

    import paper_2605_15617_b200 as prism
    import workloads as w

    torch.cuda.set_device(0)
    prism.use_torch_allocator()
    tm = w.scaled(args.config) if args.scaled else w.config(args.config)
    g = prism.Graph(tm, stream=torch.cuda.current_stream().cuda_stream, profile=True)
    for _ in range(args.reps):
        it = g.replay(args.scenarios, amp_q16=6554, kind_mask=7, algo=args.algo, record=bool(args.record))
        print(g.last_algo(), it[:2], g.last_timing(), flush=True)
    g.peak_memory()
    g.close()


if __name__ == "__main__":
    main()
