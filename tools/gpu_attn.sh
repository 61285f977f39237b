# attention rework check: GPU tests, isolated attention sweep, default bench
tag=${1:-r2e}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/${tag}_gpu.log
timeout 300 python tools/bench_attn.py > gpurun_out/${tag}_attn.txt 2>&1; echo "attn rc=$?"; cat gpurun_out/${tag}_attn.txt
timeout 1200 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/${tag}_bench.json'))
print('value %.2f tok/s'%d['value'], 'ms/step %.2f'%d['ms_per_step'], 'stages', {k:round(v,2) for k,v in d['stage_ms_per_step'].items()}, 'vanilla %.2f tok/s'%d['arms']['vanilla']['tokens_per_s'], 'e2e %.2f'%d['e2e']['value'], 'frac %.3f'%d['roofline']['frac'])"
