for v in "-DCOST5_SO=8 -DCOST5_KF=4 -DCOST5_NINC=2 -DCOST5_RI=128" "-DCOST5_SO=8 -DCOST5_KF=2 -DCOST5_NINC=1" "-DCOST5_SO=4 -DCOST5_KF=2 -DCOST5_NINC=1"; do
  echo "== $v"
  GDP_NVCC_EXTRA="$v" timeout 600 python tools/cost5_check.py 2>&1 | grep -E "C4 cost|wave|MISMATCH"
done
