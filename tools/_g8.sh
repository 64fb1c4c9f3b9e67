for v in "-DCOST5_SO=5 -DCOST5_NINC=1" "-DCOST5_SO=4" "-DCOST5_SO=6 -DCOST5_KF=2 -DCOST5_NINC=1" "-DCOST5_SO=5 -DCOST5_KF=2"; do
  GDP_NVCC_EXTRA="$v" timeout 300 python tools/cost5_time.py 1480 2>&1 | grep -E "B=|rror"
done
