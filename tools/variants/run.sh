# latency experiment: one CTA per SM (B = 148) for cost-kernel variants
for v in cur2 cur1 fused1; do
  cp tools/variants/cost4_$v.cu paper_1910_01578_b200/csrc/cost4.cu
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "variant $v"
  python tools/run_cost.py --batch 148 --reps 2 2>&1 | grep "cost 148" | tail -1
  python tools/run_cost.py --batch 256 --reps 2 2>&1 | grep "cost 256" | tail -1
done
