CS=/usr/local/cuda/bin/compute-sanitizer
$CS --tool synccheck --print-limit 3 python tools/sc_probe.py 2>&1 | grep -E "Barrier|Device Frame|SUMMARY|done" | head -12
echo ---- no PDL
ESPEC_PDL=0 $CS --tool synccheck --print-limit 3 python tools/sc_probe.py 2>&1 | grep -E "Barrier|Device Frame|SUMMARY|done" | head -12
