mkdir -p gpurun_out
for v in 0 1 0 1 0 1; do
  if [ $v = 1 ]; then export EXP_NO_CLOCKS=1; else unset EXP_NO_CLOCKS; fi
  timeout 600 python bench.py --no-cpu-baseline --no-f-rows --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('noclocks=$v', d['steps'], d['ms_per_step'], d['extra']['replay_ms_timed_steps'], d['clocks'].get('samples'))"
done > gpurun_out/exp29.txt 2>&1
