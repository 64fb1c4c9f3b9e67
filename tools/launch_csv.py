"""Summarise an ncu --csv launch list (gpu__time_duration + optional dram bytes): one line per launch."""
import csv, sys
rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
per = {}
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    key = (r[ix["ID"]], r[ix["Kernel Name"]][:40], r[ix.get("Grid Size", 0)], r[ix.get("Block Size", 0)])
    v = r[ix["Metric Value"]].replace(",", "")
    per.setdefault(key, {})[r[ix["Metric Name"]]] = (float(v) if v else 0.0, r[ix["Metric Unit"]])
for k, m in per.items():
    t = m.get("gpu__time_duration.sum", (0, ""))
    rd = m.get("dram__bytes_read.sum", (0, ""))
    wr = m.get("dram__bytes_write.sum", (0, ""))
    print(k[0], k[1], k[2], "%.1f %s" % t, "rd %.2f %s" % rd, "wr %.2f %s" % wr)
