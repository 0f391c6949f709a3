mkdir -p gpurun_out
PRISM_TRACE=1 timeout 300 python tools/exp/e2e_trace.py > gpurun_out/exp31_tr.txt 2>&1
timeout 300 python tools/exp/host_async.py > gpurun_out/exp31.txt 2>&1
for v in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --no-f-rows --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['steps'], d['ms_per_step'], d['extra']['replay_ms_timed_steps'], d['e2e']['ms_per_step'])"; done >> gpurun_out/exp31.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu >> gpurun_out/exp31.txt 2>&1
