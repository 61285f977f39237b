# round-end evidence: GPU tests, default bench (CPU leg, e2e), reference arm, launch list, full ncu of the roofline kernel
tag=${1:-r1z}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/${tag}_gpu.log
timeout 1200 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "ref rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${tag}_smoke.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgemv -s 3 -c 1 \
  -o gpurun_out/${tag}_gateup python tools/one_gemv.py 8192 57344 6 1 2 5 > gpurun_out/${tag}_gateup.log 2>&1; echo "ncu full rc=$?"
ESPEC_PROFILE_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
  --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-arms --no-cpu --e2e-tokens 0 \
  > gpurun_out/${tag}_launches.log 2>&1; echo "launches rc=$?"
