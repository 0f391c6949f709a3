mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['steps'], d['ms_per_step'], d['extra']['device_ms'], d['extra']['replay_ms_timed_steps'], d['e2e']['ms_per_step'], {k:v['replay_ms'] for k,v in d['extra']['next_rows'].items()})" > gpurun_out/exp20.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu -k "whatif or parity" >> gpurun_out/exp20.txt 2>&1
