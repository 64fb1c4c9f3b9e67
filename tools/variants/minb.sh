# k_cost4<2> (96 registers) vs k_cost4<3> (72 registers), forced through GDP_COST4_MINB: C4 (smem
# allows 2 CTAs per SM) and C3 (N ~ 20 k: smem allows 3), batch = one wave of 2 or 3 per SM;
# then the automatic choice.
for v in 2 3 ""; do
  for cb in "c4 296" "c3 296" "c3 444"; do
    set -- $cb
    echo "GDP_COST4_MINB=[$v] $1 B=$2: $(GDP_COST4_MINB=$v python tools/run_cost.py --config $1 --batch $2 --reps 3 2>&1 | grep 'cost ' | tail -1)"
  done
done
