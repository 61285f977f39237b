# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_workload.py
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for part in single tp; do
    timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_workload.py $part \
      > gpurun_out/r2_san_${tool}_${part}.log 2>&1; echo "$tool $part rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|workload done" gpurun_out/r2_san_${tool}_${part}.log | tail -3
  done
done
