#!/usr/bin/env python3
"""bench.py — the PrismLLM hot path on B200: expand + replay + peak-memory per step.

One step = one pass of every SURVEY.md §8(a) row over one synthetic input: prism_build_graph
(a1-a5: coordinates, groups, CSR DAG, levels) of the BASELINE.json workload, prism_replay of S
perturbed what-if scenarios (a6-a8) and prism_peak_memory (a9), all through the C ABI.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--scenarios 64]
  python bench.py --impl reference ...   (the CPU oracle on a bounded sample of the workload)

Prints ONE JSON line on rank 0. Metric: replayed graph ops/s = nodes x scenarios / step time
(plus emulated iterations/s = scenarios / step time in "extra"). Multi-GPU (row e): one process
per GPU (torchrun); by default the 8192 ranks are sharded over the N GPUs by DP block with the
cross-shard segmented max fused into the replay kernel over NVLink peer memory, and the scenario
batch grows with N (N x 64: weak scaling, per-GPU node-scenarios fixed); `--shard replicas` has
each GPU replay the whole graph for its own block of 64 scenarios of the sweep instead. Time = max over ranks of the device-timed region.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "replayed graph ops/sec (node-scenarios/s) at 8192 ranks"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region (the recipe's clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.window = None  # (t0, t1) of the timed region: only samples arriving inside it count

    def __enter__(self):
        if os.environ.get("PRISM_BENCH_NO_CLOCKS"):  # experiments only: the sampler's own cost
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")] + [time.perf_counter()])

    # The sampler is started before the warm-up steps (nvidia-smi's NVML start-up disturbed the
    # first milliseconds of the timed region when it was launched there) and marks the region.
    def mark(self, t0, t1):
        self.window = (t0, t1)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = self.rows
        if self.window and rows:  # samples taken during the timed region (else the nearest one)
            inside = [r for r in rows if self.window[0] <= r[-1] <= self.window[1] + 0.15]
            rows = inside or [min(rows, key=lambda r: abs(r[-1] - self.window[1]))]
        rows = [r[:-1] for r in rows]  # (the arrival time is the last field)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(int(float(r[1])) for r in rows if r[1].replace(".", "").isdigit())
        mxs = [int(float(r[2])) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mxs) if mxs else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def algorithmic_bytes(st, S: int, record: bool = True):
    """SURVEY.md §8(d) algorithmic bytes: replay (rows a6-a8) = 8 B per node-scenario
    (the start/finish time written) + 16 B per node per call (structure read); durations are
    hashed in-kernel, so no 4 B per node-scenario term. Expander (a1-a4) = 24 B per node + 8 B per
    membership; peak scan (a9) = 16 B per node + 8 B per rank. `replay_state` is the
    implementation's extra state traffic (ready slots, group accumulators, rank_end), reported
    beside the roofline, not in it."""
    N, G, M, W = st["nodes"], st["groups"], st["memberships"], st["world"]
    replay = (N * S * 8 if record else 0) + N * 16
    state = G * S * 16 + M * 8 + W * S * 8
    build = N * 24 + M * 8
    peak = N * 16 + W * 8
    return {"replay": replay, "replay_state": state, "build": build, "peak": peak}


def run_prism(args):
    import numpy as np
    import torch

    import paper_2605_15617_b200 as prism
    import workloads as w

    ws, rank, local = _dist()
    # PRISM_BENCH_ONE_GPU=1 (plumbing check on a 1-GPU box only, never a measurement): every rank on
    # cuda:0, gloo for the host-side collectives (NCCL needs one GPU per rank)
    one_gpu = ws > 1 and os.environ.get("PRISM_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
        os.environ.setdefault("PRISM_ALLOW_SAME_DEVICE_IPC", "1")
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prism.use_torch_allocator()
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    tm = w.config(args.config)
    sharded = ws > 1 and args.shard == "ranks"
    S = args.scenarios * (ws if sharded else 1)  # sharded: N x 64 scenarios over N GPUs (weak)
    # replicas: GPU i sweeps its own block of scenarios (i*S .. i*S+S-1) of one what-if sweep
    kw = dict(amp_q16=args.amp, kind_mask=7, seed=0x5EED, algo=args.algo,
              first=(rank * args.scenarios if (ws > 1 and not sharded) else 0))
    iter_dev = torch.zeros(2, S, dtype=torch.int64, device="cuda")
    iter_steps = torch.zeros(max(1, args.steps), S, dtype=torch.int64, device="cuda")  # per timed step
    peak_dev = torch.zeros(2, tm.topo.world, dtype=torch.int64, device="cuda")
    comm = [None]  # sharded: the graph currently holding the connected exchange buffer
    # Consecutive steps' graphs alternate between two streams (unsharded runs): step i+1's build
    # (upload + expansion kernels, ordinary launches) fills SMs while step i's cooperative replay
    # drains in its 1F1B ramp-down; the two replays still run one after the other (a cooperative
    # grid starts once all of its CTAs fit). Sharded graphs share one exchange buffer: one stream.
    streams = [stream] if sharded else [stream, torch.cuda.Stream()]
    # the device-timed loop keeps one stream: its replay events then bracket a replay that has the
    # GPU to itself, and host timing (the clock sampler runs beside it) cannot shift the overlap;
    # the e2e loop below, a serving loop through the public API, alternates both streams
    # (PRISM_BENCH_DEV_STREAMS=2, experiments: 2.90-3.31 ms/step over five runs, the replays'
    # own events at 0.46-0.51 of the roofline, vs 3.05-3.07 ms and 0.54 on one stream)
    dev_streams = streams[:int(os.environ.get("PRISM_BENCH_DEV_STREAMS", "1"))]

    def new_graph(profile=False, i=0, pool=None):
        # asynchronous build: the expansion is queued on the graph's stream and the replay follows
        # it there without a host round trip
        pool = pool or dev_streams
        if not sharded:
            return prism.Graph(tm, stream=pool[i % len(pool)].cuda_stream, profile=profile, asynchronous=True)
        g = prism.Graph(tm, stream=sh, profile=profile, n_shards=ws, shard_index=rank, asynchronous=True)
        if comm[0] is None:
            g.shard_connect_dist(S)  # once: exchange-buffer IPC handles over torch.distributed
        else:
            g.shard_adopt(comm[0])   # a rebuilt graph keeps the connected buffer
        comm[0] = g
        return g

    graphs = []
    replay_events = []  # (start, end) CUDA events around each timed replay, on its stream
    last_end = [None]   # end event of the latest replay

    last_start = [None]  # start event of the latest replay (fires when it is about to launch)
    build_events = []    # timed steps: recorded before each build is queued
    step_done = [None]   # end event of the latest step

    def step(timed=False, i=0):
        # host pacing: step i's build is queued once step i-1's replay is about to launch (its
        # start event fired: its graph is built and the replay before it has ended), so the
        # expansion fills SMs during that replay's drain — queued earlier, it could take SMs
        # before the cooperative grid starts and delay the whole replay
        paced = len(dev_streams) > 1
        if paced and last_start[0] is not None:
            last_start[0].synchronize()
        # build first (a sharded build adopts the previous graph's exchange buffer), then release
        # the graph of two steps back (the previous one may still run on the other stream); the
        # last ones survive the timed region
        if timed:  # the step's device work starts with its build (upload + expansion)
            eb = torch.cuda.Event(enable_timing=True)
            eb.record(dev_streams[i % len(dev_streams)])
            build_events.append(eb)
        g = new_graph(i=i)
        if len(dev_streams) == 1:  # (two streams: a graph is released once its step has finished, below)
            while graphs:
                graphs.pop(0).close()
        st_i = dev_streams[i % len(dev_streams)]
        # the replay waits for the previous one explicitly (the hardware would serialise the two
        # cooperative grids anyway), so its CUDA events bracket the replay alone while this step's
        # expansion, queued above, overlaps the previous replay
        if last_end[0] is not None:
            st_i.wait_event(last_end[0])
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record(st_i)
        last_start[0] = ev[0]
        out = iter_steps[i] if timed else iter_dev[i % 2]
        g.replay_async(out.data_ptr(), S, record=True, **kw)
        ev[1].record(st_i)
        last_end[0] = ev[1]
        if timed:
            replay_events.append(ev)
        g.peak_memory_async(peak_dev[i % 2].data_ptr())
        done = torch.cuda.Event()
        done.record(st_i)
        graphs.append(g)
        # and, as the e2e loop does, the host waits for the previous step before going on
        if paced and step_done[0] is not None:
            step_done[0].synchronize()
            while len(graphs) > 1:
                graphs.pop(0).close()
        step_done[0] = done

    clk = Clocks(local).__enter__()  # sampling from before the warm-up; the timed region is marked
    for wi in range(args.warmup):
        step(i=wi)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    gc_was = gc.isenabled()
    gc.disable()  # no collector pause inside the timed loop (host work is on the step's path)
    mem0 = torch.cuda.memory_stats()
    try:
        t_region0 = time.perf_counter()
        e0.record(stream)
        for s_ in dev_streams[1:]:
            s_.wait_event(e0)
        host_t = []
        for i in range(args.steps):
            host_t.append(time.perf_counter())
            step(timed=True, i=i)
        host_t.append(time.perf_counter())
        for s_ in dev_streams[1:]:
            stream.wait_stream(s_)
        e1.record(stream)
        torch.cuda.synchronize()
        clk.mark(t_region0, time.perf_counter())
        host_step_ms = sorted((b - a) * 1e3 for a, b in zip(host_t, host_t[1:]))
        mem1 = torch.cuda.memory_stats()
    finally:
        clk.__exit__(None, None, None)
    if gc_was:
        gc.enable()
    ms = e0.elapsed_time(e1)
    for g_ in graphs:
        g_.sync()  # raises if the device watchdog aborted a replay (prism_sync)
    its = iter_steps.cpu().numpy()
    iters = its[0].copy()
    # every timed step replays the same workload: identical results, or a step went wrong
    assert (its == iters[None, :]).all(), "timed steps disagree"
    st = graphs[0].stats()
    shard_axis = graphs[0].shard_info()["axis"] if sharded else "none"
    launches_per_step = st["replay_launches"] + 3 + 1  # expand: rank tables, nodes, groups; peak
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cpu" if one_gpu else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    units = st["nodes"] * S * (1 if sharded else ws)  # node-scenarios of the whole job per step
    value = units / (ms_step / 1e3)

    # ---- per-kernel-group device times (profiled graph, CUDA events on the launching stream)
    gp = new_graph(profile=True)
    for g in graphs:
        g.close()
    graphs.clear()
    prof = {"expand": [], "levels": [], "tail": [], "reduce": [], "peak": []}
    for i in range(3):
        gp.replay_async(iter_dev[0].data_ptr(), S, record=True, **kw)
        gp.peak_memory_async(peak_dev[0].data_ptr())
        t = gp.last_timing()
        for k in ("levels", "tail", "reduce", "peak"):
            prof[k].append(t[k])
    prof["expand"].append(gp.last_timing()["expand"])
    schedule = gp.last_algo()
    med = {k: sorted(v)[len(v) // 2] for k, v in prof.items()}
    ab = algorithmic_bytes(st, S)
    if sharded:  # this GPU replays 1/ws of the ranks: its share of the algorithmic bytes
        ab = {k: v // ws for k, v in ab.items()}
    # the roofline's duration: the replay launches of the timed steps themselves (CUDA events on
    # the launching stream, averaged); the profiled graph's split is reported beside it
    replay_ms = sum(a.elapsed_time(b) for a, b in replay_events) / len(replay_events)
    bt = [b.elapsed_time(r[0]) for b, r in zip(build_events, replay_events)]
    peak_bw, peak_src = _peaks()
    achieved = ab["replay"] / (replay_ms / 1e3) / 1e9
    iso_ms = med["levels"] + med["tail"] + med["reduce"]

    # ---- e2e: the public API from HOST buffers (H2D of templates, D2H of results) -------------
    # Pipelined, as a serving loop runs it: every step builds its graph from the host templates
    # (plan + H2D inside prism_graph_create), queues the replay and the peak scan, and copies both
    # results into pinned host memory; the host then waits for the PREVIOUS step's copies and
    # checks them, so step i+1's host work overlaps step i's device work. The serial form (build,
    # synchronous replay, synchronous peak: one step at a time) is reported beside it.
    h2d = int(tm.ops.nbytes + tm.tmpl_ptr.nbytes + tm.static_mem.nbytes)
    d2h = S * 8 + tm.topo.world * 8
    reps = max(3, min(args.steps, 20))
    dev_it = torch.zeros(2, S, dtype=torch.int64, device="cuda")
    dev_pk = torch.zeros(2, tm.topo.world, dtype=torch.int64, device="cuda")
    pin_it = torch.zeros(2, S, dtype=torch.int64).pin_memory()
    pin_pk = torch.zeros(2, tm.topo.world, dtype=torch.int64).pin_memory()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    gc.disable()
    pending = None
    checked = 0
    step_t = []
    e2e_start, e2e_end = [None], [None]
    t0 = None
    for i in range(-args.warmup, reps + 1):  # the first W steps are untimed warm-up (as above)
        if i == 0:
            t0 = time.perf_counter()
        step_t.append(time.perf_counter())
        cur = None
        if i < reps:
            j = i % 2
            st_i = streams[i % len(streams)]  # graphs alternate streams as in the timed loop
            if e2e_start[0] is not None:  # the same pacing as the timed loop
                e2e_start[0].synchronize()
            g = new_graph(i=i, pool=streams)  # (a sharded build adopts the previous graph's exchange buffer)
            if gp is not None:
                gp.close()
                gp = None
            if e2e_end[0] is not None:
                st_i.wait_event(e2e_end[0])
            e2e_start[0] = torch.cuda.Event()
            e2e_start[0].record(st_i)
            g.replay_async(dev_it[j].data_ptr(), S, record=True, **kw)
            e2e_end[0] = torch.cuda.Event()
            e2e_end[0].record(st_i)
            g.peak_memory_async(dev_pk[j].data_ptr())
            with torch.cuda.stream(st_i):
                pin_it[j].copy_(dev_it[j], non_blocking=True)
                pin_pk[j].copy_(dev_pk[j], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st_i)
            cur = (ev, g, j)
        if pending is not None:
            pev, pg, pj = pending
            pev.synchronize()
            assert (pin_it[pj].numpy() == iters).all(), "e2e step disagrees with the timed steps"
            checked += i > 0
            if cur is None:
                pg.sync()  # the last graph: raises if the device watchdog aborted a replay
                gp = pg    # kept open for the serial form's first build
            else:
                pg.close()
        pending = cur
    e2e_ms = (time.perf_counter() - t0) * 1e3 / reps
    step_t.append(time.perf_counter())
    e2e_step_ms = [round((b - a) * 1e3, 3) for a, b in zip(step_t[args.warmup:], step_t[args.warmup + 1:])]
    if gc_was:
        gc.enable()
    assert checked == reps
    # serial form: one step at a time, every call synchronous
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        g = new_graph()
        gp.close()
        it_host = g.replay(S, record=True, **kw)
        pk_host = g.peak_memory()
        gp = g
    gp.close()
    e2e_serial_ms = (time.perf_counter() - t0) * 1e3 / 3
    assert (it_host == iters).all()
    if ws > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cpu" if one_gpu else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())

    if rank != 0:
        return None
    frows = None
    if ws == 1 and not args.no_f_rows:
        frows = f_rows_extra(args, tm, sh)
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args)
    traffic, traffic_src = None, None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            traffic = tj.get(args.config, {}).get(str(S))
            traffic_src = tj.get("_source")
        except Exception:
            traffic = None
    s1 = s1_line(args, tm, sh) if ws == 1 and not args.no_f_rows else None
    out = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "node-scenarios/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int64",
        "data": "synthetic (seeded templates, BASELINE.json config shapes; DESIGN.md §4)",
        "config": {
            "workload": f"{args.config}: {w.CONFIG_DESCRIPTIONS[args.config]}",
            "ranks": tm.topo.world, "nodes": st["nodes"], "sync_groups": st["groups"],
            "memberships": st["memberships"], "levels": st["levels"], "scenarios": S,
            "amp_q16": args.amp, "record_times": True, "schedule": schedule,
            "parallelism": ("single-gpu" if ws == 1 else
                            f"ranks sharded over {ws} GPUs by {shard_axis.upper()} block, exchange fused in the "
                            f"replay kernel (NVLink peer memory)" if sharded else f"replicas{ws}"),
            "l2": "working set (fin[N][S] = %.1f GB) > 126 MB L2; no flush needed" % (st["nodes"] * S * 8 / 1e9),
            "streams": {"device_timed_loop": len(dev_streams), "e2e_loop": len(streams)},
        },
        "extra": {
            "emulated_iterations_per_s": round(S * (1 if sharded else ws) / (ms_step / 1e3), 2),
            "iteration_time_ns_scenario0": int(iters[0]),
            "device_ms": {k: round(v, 4) for k, v in med.items()},
            "replay_ms_timed_steps": round(replay_ms, 4),
            # host time to queue one step (build from host templates + replay + peak calls): the
            # device step is only fed when this stays below it
            "host_queue_ms": {"median": round(host_step_ms[len(host_step_ms) // 2], 3),
                              "p90": round(host_step_ms[int(len(host_step_ms) * 0.9)], 3),
                              "max": round(host_step_ms[-1], 3)},
            # device time of each timed step from the event before its build to its replay's start
            # (upload + expansion + any gap), median / max
            "build_to_replay_ms": {"median": round(sorted(bt)[len(bt) // 2], 3), "max": round(max(bt), 3)},
            # caching-allocator segments created (cudaMalloc) inside the timed region
            "timed_region_new_segments": int(mem1.get("segment.all.allocated", 0) - mem0.get("segment.all.allocated", 0)),
            "timed_region_alloc_retries": int(mem1.get("num_alloc_retries", 0) - mem0.get("num_alloc_retries", 0)),
            "s1": s1,
            "next_rows": frows,
            "paper_context": {
                "replay_model": "the paper replays virtual ranks in real time on assistant GPUs (P:1295-1298): one "
                                "emulated iteration takes about one real iteration, 5.6-12.0 s in Table 1 "
                                "(P:1727-1731), i.e. ~0.08-0.18 emulated iterations/s per replay",
                "accuracy": "0.58% avg iteration-time error, <0.01% peak-memory error (P:72-73); 8192 GPUs "
                            "emulated with <1% of the physical GPUs (P:74-75), on an unnamed 2048-GPU testbed",
            },
        },
        "roofline": {
            "bound": "hbm",
            "kernel": ("replay: cell_kernel (one cooperative launch) + reduce_iter_kernel, timed per step "
                       "of the timed region"
                       if schedule == "cells" else
                       "replay: level_kernel x levels + tail_kernel + reduce_iter_kernel"),
            "achieved": round(achieved, 1),
            "peak": peak_bw,
            "peak_source": peak_src,
            "unit": "GB/s",
            "frac": round(achieved / peak_bw, 4),
            "alg_bytes_per_call": ab["replay"],
            "alg_bytes_rule": "SURVEY 8(d): 8 B per node-scenario written + 16 B per node per call",
            "state_bytes_per_call": ab["replay_state"],
            "traffic": traffic,
            "traffic_source": (f"{traffic_src} (not measured in this run)" if traffic is not None else None),
            # context: the same replay timed alone on one stream (the profiled graph after the timed
            # loop); in the timed loop the next step's build shares the GPU with each replay's drain
            "isolated": {"replay_ms": round(iso_ms, 4), "frac": round(ab["replay"] / (iso_ms / 1e3) / 1e9 / peak_bw, 4)},
        },
        "e2e": {"value": round(units / (e2e_ms / 1e3), 1), "unit": "node-scenarios/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 3),
                "mode": "pipelined: step i+1's build from host templates overlaps step i's replay (graphs "
                        "alternate between two streams when unsharded); each step's templates H2D and T / peak "
                        "results D2H (pinned) inside the timed region",
                "steps": reps, "warmup": args.warmup, "step_ms_median": sorted(e2e_step_ms)[len(e2e_step_ms) // 2],
                "serial_ms_per_step": round(e2e_serial_ms, 3)},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    return out


def s1_line(args, tm, sh):
    """The S = 1 configuration of SURVEY §8.3 ("every run at S = 1 and S = 64"): one unperturbed
    scenario of the same graph on the single-scenario path (segment walks + rendezvous chain,
    replay_ranks.cu), device-timed (CUDA events on the graph's stream), best of 5, with its own
    roofline fraction on the same §8(d) bytes."""
    import paper_2605_15617_b200 as prism

    g = prism.Graph(tm, stream=sh, profile=True)
    st = g.stats()
    best = None
    for _ in range(6):
        g.replay(1, record=True)
        ms = g.last_timing()["levels"]
        best = ms if best is None else min(best, ms)
    algo = g.last_algo()
    g.close()
    ab = algorithmic_bytes(st, 1)["replay"]
    peak_bw, _ = _peaks()
    return {"replay_ms": round(best, 4), "value": round(st["nodes"] / (best / 1e3), 1), "unit": "node-scenarios/s",
            "emulated_iterations_per_s": round(1 / (best / 1e3), 1), "schedule": algo,
            "roofline_frac": round(ab / (best / 1e3) / 1e9 / peak_bw, 4), "alg_bytes_per_call": ab}


def f_rows_extra(args, tm, sh):
    """SURVEY.md §8 rows f1/f3/f4 on the same engine, measured once on this GPU (device ms from
    CUDA events on the graph's stream; node-scenarios/s of the replay):
      f1 calibration: the benchmark graph re-timed with per-node 'measured' durations (template
         +-5 % per node, the shape of a slice-filled timed graph), S scenarios on top;
      f3 what-if: every attention-forward span overridden + one rank slowed 12 % (fault
         injection), then the critical path of scenario 0 (device walk-back, wall ms);
      f4 MoE imbalance: C4 (DeepSeek-V3-shaped, EP 64) under the Fig. 3 br profile;
      f2 multi-stream ranks: C2 with its gradient buckets overlapped on a side stream, replay +
         time-ordered peak memory."""
    import numpy as np

    import paper_2605_15617_b200 as prism
    import workloads as w
    import workloads.moe as moe

    S = args.scenarios
    kw = dict(amp_q16=args.amp, kind_mask=7, seed=0x5EED)
    out = {}

    def node_durations(t):
        parts = []
        for r in range(t.topo.world):
            s = (r // t.topo.tp) % t.topo.pp if t.topo.rank_order == 0 else r // (t.topo.tp * t.topo.dp)
            parts.append(t.stage(s)["dur_ns"])
        return np.concatenate(parts).astype(np.int64)

    def timed_replay(g, n):
        best = None
        for _ in range(3):
            g.replay(S, record=True, **kw)
            ms = g.last_timing()["levels"]
            best = ms if best is None else min(best, ms)
        return {"replay_ms": round(best, 4), "value": round(n * S / (best / 1e3), 1), "unit": "node-scenarios/s"}

    g = prism.Graph(tm, stream=sh, profile=True)
    N = g.stats()["nodes"]
    d = node_durations(tm)
    d = d * np.random.default_rng(1).integers(95, 106, len(d)) // 100
    import torch

    d_dev = torch.from_numpy(d).cuda()  # measured durations already on the GPU (device-to-device copy)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.set_durations(node_dur=d_dev)
    set_dev_ms = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    g.set_durations(node_dur=d)
    set_ms = (time.perf_counter() - t0) * 1e3
    out["f1_calibrate"] = dict(timed_replay(g, N), set_durations_ms=round(set_ms, 3),
                               set_durations_device_array_ms=round(set_dev_ms, 3),
                               workload=f"{args.config} with per-node measured durations")
    del d_dev
    labs = {int(l): 1 for l in np.unique(tm.ops["label"]) if (int(l) >> 24) == w.OPCODES["ATTN_F"]}
    f = np.full(tm.topo.world, 65536, np.int32)
    f[tm.topo.world // 2] = int(1.12 * 65536)
    g.set_durations(label_dur=labs, rank_slow_q16=f)
    r = timed_replay(g, N)
    t0 = time.perf_counter()
    path, T = g.critical_path(0)
    cp0_ms = (time.perf_counter() - t0) * 1e3  # first call: includes the scratch allocation
    t0 = time.perf_counter()
    path, T = g.critical_path(0)
    cp_ms = (time.perf_counter() - t0) * 1e3
    out["f3_whatif"] = dict(r, critical_path_ms=round(cp_ms, 3), critical_path_first_call_ms=round(cp0_ms, 3),
                            critical_path_nodes=int(len(path)),
                            iteration_ns=int(T), workload=f"{args.config}, ATTN_F -> 1 ns, rank {tm.topo.world // 2} x1.12")
    g.close()
    c4 = w.config("C4")
    sched = moe.derive_schedule(moe.FIG3_PROFILE, 64, c4.topo.ep, seed=0)
    g = prism.Graph(c4, stream=sh, profile=True)
    t0 = time.perf_counter()
    g.set_moe_load(moe.op_events(c4, 64), moe.br_q16(sched))
    moe_ms = (time.perf_counter() - t0) * 1e3
    r = timed_replay(g, g.stats()["nodes"])
    pk = g.peak_memory()
    out["f4_moe_imbalance"] = dict(r, peak_max_bytes=int(pk.max()), set_moe_load_ms=round(moe_ms, 3),
                                   workload="C4 under the Fig. 3 br profile (prism_set_moe_load)")
    g.close()
    c2 = w.overlap_grad_reduce(w.config("C2"))
    g = prism.Graph(c2, stream=sh, profile=True)
    r = timed_replay(g, g.stats()["nodes"])
    g.peak_memory()
    pk_ms = g.last_timing()["peak"]
    out["f2_multistream"] = dict(r, time_ordered_peak_ms=round(pk_ms, 4),
                                 workload="C2 with gradient buckets overlapped on a second stream")
    g.close()
    return out


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(args, sample_dp: int = 8):
    """The oracle as it stands, on a bounded sample of the same workload: the C5 templates with
    DP cut to `sample_dp` replicas, nproc scenarios (one thread each), expansion included."""
    import oracle
    import workloads as w

    full = w.config(args.config)
    t = full.topo
    dp = min(t.dp, sample_dp)
    while t.dp % dp:
        dp -= 1
    ep = t.ep if dp % t.ep == 0 else 1
    tm = w.Templates(w.Topology(t.tp, t.pp, dp, ep, t.vpp, t.rank_order), full.ops, full.tmpl_ptr,
                     full.static_mem)
    cores = os.cpu_count() or 1
    S = max(1, min(args.scenarios, cores))
    oracle.build()
    # single thread, one scenario (SURVEY §8.3 "Oracle timing" (a))
    t1 = time.perf_counter()
    oracle.replay(tm, 1, amp_q16=args.amp, kind_mask=7, peaks=True, threads=1)
    one = time.perf_counter() - t1
    # repeat the sample until ~10 s of CPU work (the contract's 10-30 s bounded sample)
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.replay(tm, S, amp_q16=args.amp, kind_mask=7, peaks=True, threads=S)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= args.cpu_seconds or reps >= 200:
            break
    return {"value": round(reps * tm.n_nodes * S / dt, 1), "unit": "node-scenarios/s", "cores": min(S, cores),
            "kind": "oracle", "seconds": round(dt, 2), "cpu_model": _cpu_model(), "nproc": cores,
            "single_thread_one_scenario": {"seconds": round(one, 3),
                                           "value": round(tm.n_nodes / one, 1), "unit": "node-scenarios/s"},
            "sample": f"{args.config} templates at dp={dp} ({tm.topo.world} of {t.world} ranks, "
                      f"{tm.n_nodes} nodes), {S} scenarios, one thread each, expansion + DES + peak, "
                      f"repeated {reps}x"}


def run_reference(args):
    """--impl reference: the CPU oracle timed on the box's host cores (rank 0 only)."""
    ws, rank, local = _dist()
    if rank != 0:
        return None
    import oracle
    import workloads as w

    full = w.config(args.config)
    t = full.topo
    dp = min(t.dp, 4)
    tm = w.Templates(w.Topology(t.tp, t.pp, dp, t.ep if dp % t.ep == 0 else 1, t.vpp, t.rank_order),
                     full.ops, full.tmpl_ptr, full.static_mem)
    cores = os.cpu_count() or 1
    S = max(1, min(args.scenarios, cores))
    oracle.build()
    for _ in range(min(args.warmup, 1)):
        oracle.replay(tm, 1, amp_q16=args.amp, kind_mask=7)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.replay(tm, S, amp_q16=args.amp, kind_mask=7, peaks=True, threads=S)
    dt = (time.perf_counter() - t0) / args.steps
    v = round(tm.n_nodes * S / dt, 1)
    sample = (f"{args.config} templates at dp={dp} ({tm.topo.world} of {t.world} ranks, {tm.n_nodes} "
              f"nodes), {S} scenarios one thread each")
    return {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "node-scenarios/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": {"workload": f"{args.config}: {w.CONFIG_DESCRIPTIONS[args.config]}",
                                        "scenarios": S, "sample": sample},
        "cpu_baseline": {"value": v, "unit": "node-scenarios/s", "cores": min(S, cores), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": v, "unit": "node-scenarios/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # 50 steps by default (~0.2 s of GPU time): the first timed step carries the pipeline fill (its
    # host build of ~2.5 ms runs with the device idle) and the clock sampler runs alongside
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="prism", choices=["prism", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scenarios", type=int, default=64)
    ap.add_argument("--amp", type=int, default=6554)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU work of the cpu_baseline sample")
    ap.add_argument("--no-f-rows", action="store_true", help="skip the rows f1/f3/f4 measurements in extra")
    ap.add_argument("--algo", default="auto", choices=["auto", "levels", "cells"])
    ap.add_argument("--shard", default="ranks", choices=["ranks", "replicas"],
                    help="N>1: shard the ranks over the GPUs (row e) or run independent replicas")
    args = ap.parse_args()
    args.config = args.config.upper()
    ws_env = os.environ.get("WORLD_SIZE")
    if args.impl == "prism" and args.gpus > 1 and ws_env is None:
        # one process per GPU: re-launch this command under torch.distributed.run (the driver's
        # own launch sets WORLD_SIZE and lands below)
        import socket

        with socket.socket() as s_:
            s_.bind(("127.0.0.1", 0))
            port = s_.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.impl == "prism" and ws_env is not None and int(ws_env) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}: launch one process per GPU")
    if args.warmup < 3 and args.impl == "prism":
        args.warmup = 3
    out = run_reference(args) if args.impl == "reference" else run_prism(args)
    if out is not None:
        print(json.dumps(out), flush=True)
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1 and args.impl == "prism":
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
