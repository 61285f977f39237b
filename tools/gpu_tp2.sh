# functional check of the N>1 bench path on a 1-GPU box: two ranks on cuda:0
# (timings meaningless), drafter tensor-parallel and layer-parallel; then the
# TP-N shard proxies (per-GPU step time at TP-N shard shapes)
tag=${1:-tp2}
mkdir -p gpurun_out
for layout in tp lp; do
  ESPEC_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --workload mini --no-cpu \
    --e2e-tokens 16 --draft-layout $layout > gpurun_out/${tag}_mini_${layout}.json 2> gpurun_out/${tag}_mini_${layout}.err
  echo "tp2 $layout rc=$?"; head -c 400 gpurun_out/${tag}_mini_${layout}.json; echo; tail -2 gpurun_out/${tag}_mini_${layout}.err
done
for N in 8 4 2; do for layout in tp lp; do
  timeout 900 python bench.py --tp-proxy $N --draft-layout $layout --no-cpu --e2e-tokens 0 \
    > gpurun_out/${tag}_proxy${N}_${layout}.json 2> gpurun_out/${tag}_proxy${N}_${layout}.err; echo "proxy $N $layout rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/${tag}_proxy${N}_${layout}.json'))
print('TP-$N proxy ($layout drafter): ms/step %.2f'%d['ms_per_step'], 'stages', {k:round(v,2) for k,v in d['stage_ms_per_step'].items()}, 'vanilla ms %.2f'%d['arms']['vanilla']['ms_per_step'], 'sd ms %.2f'%d['arms']['sd']['ms_per_step'], 'sd draft ms/token %.2f'%d['arms']['sd']['draft_ms_per_token'], 'es draft ms/token %.2f'%d['draft_ms_per_token'])"
done; done
