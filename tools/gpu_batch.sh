# Cost-kernel grid sizing: the C4 step at B = 256 / 296 (= 148 SMs x 2 resident CTAs) / 592, and
# the GPU tests of this build.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for B in 256 296 592; do
  timeout 600 python bench.py --batch $B --steps 5 --warmup 3 --no-cpu-baseline --no-kernels > gpurun_out/bench_b$B.json 2> gpurun_out/bench_b$B.err
  head -c 400 gpurun_out/bench_b$B.json; echo
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
