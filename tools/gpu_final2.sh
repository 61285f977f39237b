# round-end evidence + in-stream site times: tools/gpu_final.sh, then tools/site_times.py
tag=${1:-r2z}
bash tools/gpu_final.sh $tag
timeout 600 python tools/site_times.py > gpurun_out/${tag}_sites.txt 2>&1; echo "sites rc=$?"; cat gpurun_out/${tag}_sites.txt | tail -5
python tools/ncu_summary.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches_summary.txt 2>&1; head -12 gpurun_out/${tag}_launches_summary.txt
