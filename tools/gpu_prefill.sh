timeout 600 python tools/prefill_profile.py 512 2>&1 | tail -1
ESPEC_PROFILE_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
  --csv --log-file gpurun_out/prefill_launches.csv python tools/prefill_profile.py 512 > gpurun_out/prefill_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/prefill_launches.csv | head -25
