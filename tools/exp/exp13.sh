mkdir -p gpurun_out
for n in 20 20 50; do timeout 600 python bench.py --no-cpu-baseline --no-f-rows --steps $n 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['steps'], d['ms_per_step'], d['extra']['device_ms'], d['extra']['replay_ms_timed_steps'])"; done > gpurun_out/exp13.txt 2>&1
