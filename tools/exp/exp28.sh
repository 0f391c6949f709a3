mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-f-rows > gpurun_out/exp28_ncu.csv 2>&1
python tools/exp/fast_sweep.py 4,32,256 4,32,256 > gpurun_out/exp28.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-f-rows --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['steps'], d['ms_per_step'], d['extra']['device_ms'], d['extra']['replay_ms_timed_steps'])" >> gpurun_out/exp28.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu -k "csr or parity or whatif" >> gpurun_out/exp28.txt 2>&1
