timeout 900 python -m pytest tests/test_gpu_tp.py tests/test_gpu_tp_ipc.py -x -q 2>&1 | tail -3
for N in 8 2; do
  timeout 900 python bench.py --tp-proxy $N --no-cpu --e2e-tokens 0 > gpurun_out/fz_proxy$N.json 2> gpurun_out/fz_proxy$N.err; echo "proxy $N rc=$?"; tail -2 gpurun_out/fz_proxy$N.err
  python -c "
import json; d=json.load(open('gpurun_out/fz_proxy$N.json'))
print('TP-$N proxy: ms/step %.2f'%d['ms_per_step'], 'stages', {k:round(v,2) for k,v in d['stage_ms_per_step'].items()}, 'vanilla ms %.2f'%d['arms']['vanilla']['ms_per_step'], 'sd ms %.2f'%d['arms']['sd']['ms_per_step'])"
done
