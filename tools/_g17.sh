python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 python tools/cost5_time.py 1480 1776 2>&1 | grep "B="
GDP_NVCC_EXTRA="-DCOST5_MINB=10" timeout 600 python tools/cost5_time.py 1480 2>&1 | grep "B="
timeout 900 python tools/cost5_check.py 2>&1 | grep -v "^C4 cost" | tail -6
