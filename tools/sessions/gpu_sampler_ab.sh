# A/B: does the nvidia-smi clock sampler perturb the config-2 step? main loop only, 5 steps, alternating
for r in 1 2 3; do
  python bench.py --no-sub --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/s_on_$r.json 2>&1
  python bench.py --no-sub --no-e2e --no-cpu-baseline --steps 5 --no-clocks > gpurun_out/s_off_$r.json 2>&1
done
for f in gpurun_out/s_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],1), d['step_ms_rank0'], d['create_ms_rank0'])"; done
