"""Aggregate an ncu source page (cuda,sass CSV) per CUDA line: stall samples and instructions."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, src = {}, {}
fname = "?"
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[2] != "-":
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    key_ = (fname, ln)
    agg[key_] = (float(r[4] or 0), float(r[7] or 0))
    src[key_] = r[1]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print("samples", ts, "warp-instructions", ti)
key = 1 if (len(sys.argv) > 3 and sys.argv[3] == "inst") else 0
for ln, (s, i) in sorted(agg.items(), key=lambda x: -x[1][key])[:n]:
    print("%-22s %5d %6.2f%%smp %6.2f%%ins  %s" % (ln[0][:22], ln[1], 100 * s / ts, 100 * i / ti, src[ln][:80]))
