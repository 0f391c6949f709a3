mkdir -p gpurun_out
for v in 1 2 3 4 5; do
  timeout 600 python bench.py --no-cpu-baseline --no-f-rows --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['steps'], d['ms_per_step'], d['extra']['replay_ms_timed_steps'], d['e2e']['ms_per_step'])"
done > gpurun_out/exp30.txt 2>&1
