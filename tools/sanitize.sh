#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck of the replay kernels on small graphs
mkdir -p gpurun_out
cat > /tmp/san_case.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_15617_b200 as prism, workloads as w, oracle
torch.cuda.set_device(0); prism.use_torch_allocator()
s = torch.cuda.current_stream().cuda_stream
for tm, S in ((w.config("C1"), 64), (w.random_templates(3, max_world=16, max_ops=30), 33),
              (w.random_templates(5, max_world=16, max_ops=30, streams=2), 5), (w.scaled("C4"), 40)):
    g = prism.Graph(tm, stream=s)
    it = g.replay(S, amp_q16=6554, kind_mask=7)
    assert np.array_equal(it, oracle.replay(tm, S, amp_q16=6554, kind_mask=7, peaks=False)["iter"])
    g.peak_memory(); g.replay(1, amp_q16=6554, kind_mask=7)
    g.close()
tm = w.scaled("C2")
gs = [prism.Graph(tm, stream=s, n_shards=2, shard_index=i) for i in range(2)]
for g in gs: g.shard_prepare(32)
for g in gs: g.shard_connect_local(gs)
out = torch.zeros(32, dtype=torch.int64, device="cuda")
prism.replay_local_shards(gs, out.data_ptr(), 32, amp_q16=6554, kind_mask=7)
torch.cuda.synchronize(); gs[0].sync()
assert np.array_equal(out.cpu().numpy(), oracle.replay(tm, 32, amp_q16=6554, kind_mask=7, peaks=False)["iter"])
print("case ok")
PY
for tool in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_case.py > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.log
done
