# Register cap for three resident k_cost4 CTAs per SM: C4 (smem allows 2 per SM) and C3
# (N ~ 20 k: smem allows 3 per SM), batch = one wave of 2 or 3 CTAs per SM.
for v in "" "-DCOST4_MINB=3"; do
  GDP_NVCC_EXTRA="$v" python -c "from paper_1910_01578_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || echo "build failed: $v"
  for cb in "c4 296" "c3 296" "c3 444"; do
    set -- $cb
    echo "variant [$v] $1 B=$2: $(python tools/run_cost.py --config $1 --batch $2 --reps 3 2>&1 | grep 'cost ' | tail -1)"
  done
done
