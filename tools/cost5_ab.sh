# A/B of k_cost5 compile-time variants at the C4 wave: tools/cost5_ab.sh "<flags A>" "<flags B>" ...
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "$@"; do
  GDP_NVCC_EXTRA="$v" timeout 600 python tools/cost5_time.py ${B:-2368} 2>&1 | grep "B="
done
