# TP-N shard proxy: rank 0 of a TP-N group alone on one GPU (collectives loop back)
tag=${1:-r2tp}
mkdir -p gpurun_out
for N in 8 4 2; do
  timeout 900 python bench.py --tp-proxy $N --no-cpu --e2e-tokens 0 > gpurun_out/${tag}_proxy${N}.json 2> gpurun_out/${tag}_proxy${N}.err; echo "proxy $N rc=$?"; tail -2 gpurun_out/${tag}_proxy${N}.err
  python -c "
import json; d=json.load(open('gpurun_out/${tag}_proxy${N}.json'))
print('TP-$N proxy: ms/step %.2f'%d['ms_per_step'], 'stages', {k:round(v,2) for k,v in d['stage_ms_per_step'].items()}, 'vanilla ms %.2f'%d['arms']['vanilla']['ms_per_step'], 'sd ms %.2f'%d['arms']['sd']['ms_per_step'], 'launches', d['gpu_launches'], 'stage_roofline', {k:(round(v,2) if v else v) for k,v in d['stage_roofline'].items() if k!='unit'})"
done
