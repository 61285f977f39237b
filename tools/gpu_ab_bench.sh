# same-box A/B of the C2 bench: this build vs paper_2502_02493_b200/libespec_ab.so
# (tools/build_ab.sh), alternating, 10 timed steps each -> gpurun_out/<tag>_bench.txt
tag=${1:-ab}; reps=${2:-3}
mkdir -p gpurun_out
for i in $(seq $reps); do for lib in libespec_ab.so libespec_b200.so; do
  echo "== $lib"; ESPEC_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-arms 2>/dev/null | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); s=j.get('stage_ms_per_step') or {}
print(f\"{j['value']:.3f} tok/s {j['ms_per_step']:.2f} ms/step e2e {j['e2e']['value']:.3f}\", {k: round(v, 2) for k, v in s.items()} if isinstance(s, dict) else s)"
done; done > gpurun_out/${tag}_bench.txt 2>&1; cat gpurun_out/${tag}_bench.txt
