for v in "" "-DWG_MAJ=0" "-DWG_SWAP"; do
  echo "=== variant [$v]"
  GDP_NVCC_EXTRA="$v" python tools/wgrad_probe.py 2>&1 | grep -A3 "^dWo"
done
