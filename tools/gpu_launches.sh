tag=${1:-r1e}
ESPEC_PROFILE_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
  --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-arms --no-cpu --e2e-tokens 0 \
  > gpurun_out/${tag}_launches.log 2>&1; echo "launches rc=$?"
python tools/ncu_summary.py gpurun_out/${tag}_launches.csv | head -30
