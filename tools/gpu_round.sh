#!/bin/bash
# One gpurun pass: GPU parity tests, default bench, launch list, full ncu of the roofline kernel.
# usage (under gpurun): bash tools/gpu_round.sh [tag]
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
ESPEC_PROFILE_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
  --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-arms --no-cpu --e2e-tokens 0 \
  > gpurun_out/${tag}_launches.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgemv -s 3 -c 1 \
  -o gpurun_out/${tag}_gateup python tools/one_gemv.py 8192 57344 6 1 2 5 > gpurun_out/${tag}_gateup.log 2>&1; echo "ncu full rc=$?"
