# A/B of cost-kernel variants in one session (C4, B = 256)
for rep in 1 2; do
for v in head clean; do
  cp tools/variants/cost4_$v.cu paper_1910_01578_b200/csrc/cost4.cu
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "variant $v: $(python tools/run_cost.py --batch 256 --reps 3 2>&1 | grep 'cost 256' | tail -1)"
done
done
