mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_megakernel.py -x -q 2>&1 | tail -2
for pf in 0 256 512 768 1024; do
  ESPEC_MK_PF_KB=$pf timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --e2e-tokens 0 > gpurun_out/pf_$pf.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pf_$pf.json'))
print('pf=$pf', 'ms/step %.2f'%d['ms_per_step'], 'stages', {k:round(v,2) for k,v in d['stage_ms_per_step'].items()}, 'vanilla ms %.2f'%d['arms']['vanilla']['ms_per_step'], 'sd ms %.2f'%d['arms']['sd']['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])"
done
