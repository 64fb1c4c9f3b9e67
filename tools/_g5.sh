python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest -q tests/test_gpu_dist.py tests/test_gpu_train.py 2>&1 | tail -4
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 1000000 python tools/sanitize.py small > gpurun_out/san_racecheck_full.log 2>&1
grep -E "^=========\s+(Error|Warning)" -A2 gpurun_out/san_racecheck_full.log | grep -oE "(Error|Warning): \(?[A-Za-z ]*\)? ?[A-Za-z]* hazard|k_[a-z_0-9]+(<[0-9]+>)?\(|[a-z_0-9]+\.cu:[0-9]+" | paste - - - 2>/dev/null | sort | uniq -c | sort -rn | head -30 > gpurun_out/san_racecheck_summary.txt
cat gpurun_out/san_racecheck_summary.txt
grep "RACECHECK SUMMARY" gpurun_out/san_racecheck_full.log
rm -f gpurun_out/san_racecheck_full.log
