mkdir -p gpurun_out
for n in 20 20 40; do timeout 600 python bench.py --no-cpu-baseline --steps $n 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['steps'], d['ms_per_step'], d['extra']['device_ms'], d['extra']['replay_ms_timed_steps'], d['e2e']['ms_per_step'], {k:v['replay_ms'] for k,v in d['extra']['next_rows'].items()})"; done > gpurun_out/exp19.txt 2>&1
timeout 300 python tools/exp/host_async.py >> gpurun_out/exp19.txt 2>&1
