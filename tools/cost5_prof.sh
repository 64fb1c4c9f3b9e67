for B in 1 148 2368; do
  echo "== B=$B"
  GDP_NVCC_EXTRA="-DCOST5_PROF" timeout 600 python tools/run_cost.py --batch $B --reps 1 2>&1 | grep -E "C5PROF|C5MEM" | head -2
done
