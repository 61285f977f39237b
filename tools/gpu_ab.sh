# A/B: megakernel on/off on the C2 bench (no CPU leg)
for mk in 1 0; do
  ESPEC_MK=$mk timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu --e2e-tokens 0 > gpurun_out/ab_$mk.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_$mk.json'))
print('mk=$mk', 'ms/step %.2f'%d['ms_per_step'], 'stages', {k:round(v,2) for k,v in d['stage_ms_per_step'].items()}, 'vanilla ms %.2f'%d['arms']['vanilla']['ms_per_step'], 'sd ms %.2f'%d['arms']['sd']['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'launches', d['gpu_launches'])"
done
