# A/B over env settings on the C2 bench (no CPU leg): bash tools/gpu_ab.sh "ENV1" "ENV2" ...
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu --e2e-tokens 0 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$cfg', 'ms/step %.2f'%d['ms_per_step'], 'stages', {k:round(v,2) for k,v in d['stage_ms_per_step'].items()}, 'vanilla ms %.2f'%d['arms']['vanilla']['ms_per_step'], 'sd ms %.2f'%d['arms']['sd']['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])"
done
