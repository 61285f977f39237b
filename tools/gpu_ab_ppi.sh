# C2 bench A/B over the attention chunk size (pages per CTA) at ctx 512
tag=${1:-ppi}
mkdir -p gpurun_out
for i in 1 2 3; do for e in "ESPEC_ATTN_PPI=2" "ESPEC_ATTN_PPI=3" "ESPEC_ATTN_PPI=4"; do
  echo "== $e"; env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-arms 2>/dev/null | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms_per_step') or {}
print(f\"{j['value']:.3f} tok/s {j['ms_per_step']:.2f} ms/step e2e {j['e2e']['value']:.3f}\", {k: round(v, 2) for k, v in s.items()})"
done; done > gpurun_out/${tag}_bench.txt 2>&1; cat gpurun_out/${tag}_bench.txt
