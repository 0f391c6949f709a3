mkdir -p gpurun_out
PRISM_TRACE=1 python -c "
import sys; sys.path.insert(0, '.')
import torch, paper_2605_15617_b200 as prism, workloads as w
torch.cuda.set_device(0); prism.use_torch_allocator(); tm = w.config('C5')
prev = None
for i in range(12):
    g = prism.Graph(tm, asynchronous=True)
    if prev: prev.close()
    prev = g
torch.cuda.synchronize()
" 2> gpurun_out/trace.log
