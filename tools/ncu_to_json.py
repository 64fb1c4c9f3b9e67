"""Summarise one ncu --set full capture of the cost kernel into profiles/cost_kernel_ncu.json
(read by bench.py for the issue-slot roofline and the DRAM traffic of the dominant kernel)."""
import csv, json, subprocess, sys
rep, out, kernel, workload, batch, source = sys.argv[1:7]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
f = lambda k: float(d[k].replace(",", ""))
res = {
    "source": source,
    "kernel": kernel,
    "workload": workload,
    "batch": int(batch),
    "warp_inst_per_launch": int(f("smsp__inst_executed.sum")),
    "dram_bytes_read_per_launch": int(f("dram__bytes_read.sum") * (1e6 if d.get("dram__bytes_read.sum") and h else 1)),
    "ncu_duration_ms": f("gpu__time_duration.sum"),
    "smsp_issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "sm_warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
}
units = dict(zip(h, rows[1]))
def to_bytes(k):
    u = units.get(k, "byte")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
    return int(f(k) * scale)
res["dram_bytes_read_per_launch"] = to_bytes("dram__bytes_read.sum")
res["dram_bytes_write_per_launch"] = to_bytes("dram__bytes_write.sum")
dur_unit = units.get("gpu__time_duration.sum", "msecond")
res["ncu_duration_ms"] = f("gpu__time_duration.sum") * {"msecond": 1, "usecond": 1e-3, "nsecond": 1e-6, "second": 1e3}.get(dur_unit, 1)
# warp-state breakdown: cycles a warp spends per issued instruction, by stall reason
st = {}
for k in h:
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        x = f(k)
        if x >= 0.05:
            st[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(x, 3)
if st:
    res["stall_cycles_per_issued_inst"] = dict(sorted(st.items(), key=lambda kv: -kv[1]))
    res["warp_latency_per_inst"] = round(f("smsp__average_warp_latency_per_inst_issued.ratio"), 3)
json.dump(res, open(out, "w"), indent=2)
print(json.dumps(res, indent=2))
