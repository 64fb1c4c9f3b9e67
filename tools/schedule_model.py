"""Schedule model of the cost kernel's parallelism on one C4 placement (uses the oracle's
start times; host only).  Prints: distinct event ticks; static windows of L ticks; the
critical path of an ideal asynchronous conservative simulator (an event on device q at tau
waits for device q's previous event and for every other device's events at <= tau - L);
dynamic-horizon window counts.  DESIGN.md §7 "What bounds it"."""
import bisect, collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads
from oracle import simulate as S

W = workloads.config("c4", batch=4)
g = W.graphs[0]
topo = workloads.topology(g, W.d)
D = np.random.default_rng(0).integers(0, W.d, size=(1, g.N)).astype(np.uint8)
r = S.simulate_batch(g, topo, D, want_start=True)
st = r["start"]
dur = g.compute_cost * topo.speed[D[0]]
fin = st + dur
dev = D[0]
e = g.edges
u, w = e[:, 0], e[:, 1]
cross = dev[u] != dev[w]
arr = fin[u[cross]] + (g.output_bytes[u[cross]] + 9999) // 10000 + 5   # no channel queueing
ev = collections.defaultdict(collections.Counter)
for v in range(g.N):
    ev[int(fin[v])][(int(dev[v]), "f")] += 1
    ev[int(st[v])][(int(dev[v]), "s")] += 1
for a_, w_ in zip(arr.tolist(), w[cross].tolist()):
    ev[int(a_)][(int(dev[w_]), "a")] += 1
T = sorted(ev)
print("N", g.N, "makespan", int(r["makespan"][0]), "distinct event ticks", len(T))
Lat = int(os.environ.get("LAT", "5"))
i = nw = 0
while i < len(T):
    t0 = T[i]; nw += 1
    while i < len(T) and T[i] < t0 + Lat:
        i += 1
print("static windows (L = %d):" % Lat, nw)
per = collections.defaultdict(set)
for t_, cn in ev.items():
    for (dv, kd), c in cn.items():
        per[dv].add(t_)
per = {k: sorted(v) for k, v in per.items()}
done = {q: [0] * len(ts) for q, ts in per.items()}
idx = {q: 0 for q in per}
for t_, q in sorted((t_, q) for q, ts in per.items() for t_ in ts):
    k_ = idx[q]; idx[q] += 1
    m = done[q][k_ - 1] if k_ > 0 else 0
    for k, ts in per.items():
        if k != q:
            j = bisect.bisect_right(ts, t_ - Lat) - 1
            if j >= 0:
                m = max(m, done[k][j])
    done[q][k_] = m + 1
print("async critical path (local instants):", max(max(v) for v in done.values()),
      " local instants total", sum(len(v) for v in per.values()))
ops = collections.defaultdict(list)
for v in range(g.N):
    ops[int(dev[v])].append((int(st[v]), int(fin[v])))
starts = {k: sorted(a for a, _ in ops[k]) for k in ops}
for k in ops:
    ops[k].sort()
def dyn(optimistic, WM):
    i = nw = 0
    while i < len(T):
        t0 = T[i]; nw += 1
        H = t0 + WM
        for k in range(W.d):
            ss = starts[k]; j = bisect.bisect_right(ss, t0) - 1
            if j >= 0 and ops[k][j][1] >= t0:
                e_ = ops[k][j][1] + Lat
            else:
                jn = bisect.bisect_left(ss, t0)
                ns = ss[jn] if jn < len(ss) else 10 ** 12
                e_ = (max(t0, ns) if optimistic else t0) + 1 + Lat
            H = min(H, e_)
        while i < len(T) and T[i] < H:
            i += 1
    return nw
for WM in (8, 16):
    print("dynamic windows, cap", WM, ": optimistic", dyn(True, WM), " pessimistic", dyn(False, WM))

# two-phase windows: events at T0 first, then (T0, H) with H = min over devices of the earliest
# possible new push after phase 1 (running: fin + L; idle: next start + 1 + L, where next start is
# the true one (optimistic) or T0 + 1 (pessimistic)); cost = sum over windows of the busiest
# device's local instants (+1 for phase 1)
def two_phase(optimistic, WM=64):
    i = nw = 0
    crit = 0
    fins = {k: sorted(f for _, f in ops[k]) for k in ops}
    while i < len(T):
        t0 = T[i]; nw += 1
        H = t0 + WM
        for k in range(W.d):
            ff = fins[k]; j = bisect.bisect_right(ff, t0)          # first finish after t0
            ss = starts[k]; js = bisect.bisect_right(ss, t0) - 1
            running = js >= 0 and ops[k][js][1] > t0
            if running:
                e_ = ops[k][js][1] + Lat
            else:
                jn = bisect.bisect_right(ss, t0)
                ns = ss[jn] if jn < len(ss) else 10 ** 12
                e_ = (ns if optimistic else t0 + 1) + 1 + Lat
            H = min(H, e_)
        per_dev = collections.Counter()
        while i < len(T) and T[i] < H:
            for (dv, kd) in ev[T[i]]:
                per_dev[dv] += 1 if kd != "s" else 0
            i += 1
        crit += max(per_dev.values()) if per_dev else 0
    return nw, crit
print("two-phase windows (optimistic, pessimistic):", two_phase(True), two_phase(False))
i = nw = crit = 0
while i < len(T):
    t0 = T[i]; nw += 1
    per_dev = collections.Counter()
    while i < len(T) and T[i] < t0 + Lat:
        for (dv, kd) in ev[T[i]]:
            per_dev[dv] += 1 if kd != "s" else 0
        i += 1
    crit += max(per_dev.values()) if per_dev else 0
print("static windows, critical local events:", nw, crit)
