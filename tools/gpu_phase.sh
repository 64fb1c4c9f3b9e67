python -c "import __graft_entry__ as g; g.build()" 
for c in c1 c2 c4; do timeout 900 python bench.py --train --config $c --steps 3 --warmup 1 2>/dev/null | tail -1; done
