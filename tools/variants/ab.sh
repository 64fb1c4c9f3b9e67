# A/B of compile-time variants of the cost kernel in one GPU session (C4, B = 256):
#   bash tools/variants/ab.sh "-DA=1" "-DB=2" ...   (each argument = GDP_NVCC_EXTRA of one build)
for rep in 1 2; do
for v in "$@"; do
  GDP_NVCC_EXTRA="$v" python -c "from paper_1910_01578_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || echo "build failed: $v"
  echo "variant [$v]: $(python tools/run_cost.py --batch 256 --reps 3 2>&1 | grep 'cost 256' | tail -1)"
done
done
