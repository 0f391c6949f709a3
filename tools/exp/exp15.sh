mkdir -p gpurun_out
timeout 300 python tools/exp/host_async.py > gpurun_out/exp15_host.txt 2>&1
timeout 300 python tools/step_timeline.py > gpurun_out/exp15_tl.txt 2>&1
for n in 20 20; do timeout 600 python bench.py --no-cpu-baseline --no-f-rows --steps $n 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['steps'], d['ms_per_step'], d['extra']['device_ms'], d['extra']['replay_ms_timed_steps'], d['e2e']['ms_per_step'])"; done > gpurun_out/exp15_bench.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/exp15_pytest.txt 2>&1
