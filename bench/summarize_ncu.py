"""Summarise a bench ncu pass (bench/ncu_bench.sh) into profiles/: the launch list's per-kernel
share of the step and the full capture's key counters; writes profiles/traffic.json (DRAM bytes
per launch of the dominant kernel, the `roofline.traffic` field of bench.py).
Usage: python bench/summarize_ncu.py r01"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1] if len(sys.argv) > 1 else "r01"
G = os.path.join(ROOT, "gpurun_out")


def rows(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    return list(csv.DictReader(io.StringIO(txt[i:])))


launch = {}
for r in rows(os.path.join(G, f"{R}_launches_bench.csv")):
    k = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
    v = float(r["Metric Value"].replace(",", ""))
    d = launch.setdefault((int(r["ID"]), k), {})
    d[r["Metric Name"]] = v
per = {}
for (i, k), d in launch.items():
    e = per.setdefault(k, dict(n=0, us=0.0, dram=0.0))
    e["n"] += 1
    e["us"] += d.get("gpu__time_duration.sum", 0) / 1e3
    e["dram"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
tot = sum(e["us"] for e in per.values())
lst = {k: dict(launches=e["n"], us_per_launch=round(e["us"] / e["n"], 2), share=round(e["us"] / tot, 4),
               dram_MB_per_launch=round(e["dram"] / e["n"] / 1e6, 2)) for k, e in per.items()}

full = rows(os.path.join(G, f"{R}_full_bench_raw.csv"))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
summary = {}
if full:
    r = full[-1]
    hdr = list(r.keys())
    for k in keys:
        m = [h for h in hdr if h.startswith(k)]
        if m:
            summary[k] = r[m[0]]
    summary["kernel"] = r.get("Kernel Name", "")[:120]
out = dict(round=R, launch_list=lst, full_capture=summary)
json.dump(out, open(os.path.join(ROOT, "profiles", f"{R}_ncu_bench.json"), "w"), indent=1)
if summary.get("dram__bytes_read.sum"):
    def num(s):
        return float(str(s).replace(",", ""))
    traffic = num(summary["dram__bytes_read.sum"]) + num(summary.get("dram__bytes_write.sum", 0))
    json.dump({"tc_spmv_tile[0]": traffic, "source": f"profiles/{R}_ncu_bench.json (ncu --set full, bytes)"},
              open(os.path.join(ROOT, "profiles", "traffic.json"), "w"))
print(json.dumps(out, indent=1))
