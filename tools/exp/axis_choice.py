import sys; sys.path.insert(0, '.')
import torch, paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator()
for name in ("C2", "C3", "C4", "C5"):
    tm = w.config(name)
    for n in (2, 4, 8):
        g = prism.Graph(tm, n_shards=n, shard_index=0)
        print(name, n, g.shard_info()); g.close()
