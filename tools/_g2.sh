GDP_NVCC_EXTRA=-DCOST5_PROF timeout 300 python tools/run_cost.py --batch 296 --reps 1 > gpurun_out/c5prof296.log 2>&1
GDP_NVCC_EXTRA=-DCOST5_PROF timeout 300 python tools/run_cost.py --batch 1 --reps 1 > gpurun_out/c5prof1.log 2>&1
GDP_NVCC_EXTRA=-DCOST5_PROF timeout 300 python tools/run_cost.py --batch 592 --reps 1 > gpurun_out/c5prof592.log 2>&1
grep -h "C5\|cost" gpurun_out/c5prof*.log
