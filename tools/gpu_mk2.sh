mkdir -p gpurun_out
tag=${1:-r1d}
timeout 600 python -m pytest tests/test_gpu_megakernel.py -x -q > gpurun_out/${tag}_mk.log 2>&1; rc=$?; echo "mk rc=$rc"; tail -3 gpurun_out/${tag}_mk.log
timeout 900 python bench.py --no-cpu --e2e-tokens 0 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"; head -c 1500 gpurun_out/${tag}_bench.json; tail -3 gpurun_out/${tag}_bench.err
ESPEC_PROFILE_REGION=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:decode_mk -s 5 -c 1 \
  -o gpurun_out/${tag}_mkbase python bench.py --steps 1 --warmup 3 --no-arms --no-cpu --e2e-tokens 0 > gpurun_out/${tag}_mkbase.log 2>&1; echo "ncu rc=$?"
