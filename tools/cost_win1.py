"""One case of tools/cost_win.py for ncu: isolated ops on device 0, cost 1 (five local instants
per window) or 1000 (one)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.cost_win import run
c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
chain = len(sys.argv) > 2 and sys.argv[2] == "chain"
d = int(sys.argv[3]) if len(sys.argv) > 3 else 8
print("ms", run(20000, c, d=d, chain=chain))
