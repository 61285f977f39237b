# prefill A/B: this build vs paper_2502_02493_b200/libespec_ab.so (tools/build_ab.sh), alternating,
# then the prefill / bf16-shape parity tests on this build -> gpurun_out/<tag>_*
tag=${1:-pre}
mkdir -p gpurun_out
for lib in libespec_ab.so libespec_b200.so libespec_ab.so libespec_b200.so; do
  echo "== $lib"; ESPEC_LIB=$lib timeout 600 python tools/prefill_profile.py 512 2>&1 | tail -1
done > gpurun_out/${tag}_time.txt 2>&1; cat gpurun_out/${tag}_time.txt
timeout 1200 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_bf16_shapes.py tests/test_gpu_parity.py -x -q > gpurun_out/${tag}_tests.txt 2>&1; tail -3 gpurun_out/${tag}_tests.txt
ESPEC_PROFILE_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
  --csv --log-file gpurun_out/${tag}_launches.csv python tools/prefill_profile.py 512 > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches.txt 2>&1; head -14 gpurun_out/${tag}_launches.txt
