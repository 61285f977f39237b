# r2: smoke (fp32 + bf16 perf path), default bench, reference arm, ncu dram bytes of the c3/c4 gate/up launches
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2b_smoke.log
timeout 1200 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/r2b_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err; echo "ref rc=$?"; head -c 600 gpurun_out/r2b_ref.json
for shp in "8192 59136 c3" "5120 55296 c4"; do set -- $shp
timeout 600 ncu --set full --clock-control none -k regex:sgemv -s 3 -c 1 -o gpurun_out/r2b_gateup_$3 python tools/one_gemv.py $1 $2 6 1 2 5 > gpurun_out/r2b_gateup_$3.log 2>&1; echo "ncu $3 rc=$?"
done
