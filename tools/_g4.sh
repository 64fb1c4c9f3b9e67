mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
for tool in memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/san_$tool.log
done
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize.py small > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -6 gpurun_out/san_racecheck.log
