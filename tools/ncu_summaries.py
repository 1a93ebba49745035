#!/usr/bin/env python
"""Summarise ncu outputs into the JSON files committed under profiles/.

    python tools/ncu_summaries.py launches <launches.csv> <out.json> <about>
    python tools/ncu_summaries.py full <report.ncu-rep> <out.json> <about> [traffic-key]
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct"]


OURS = ("fused_kernel", "average_kernel", "tma_kernel", "peer_kernel", "peer_tma_kernel", "peer_ws_kernel",
        "avg_publish_kernel", "avg_publish_tma_kernel", "copy_tensors_kernel", "checksum_kernel", "fill_u64_kernel")


def short(name):
    if "at::cuda" in name or "spin_kernel" in name:
        return "torch: " + name.split("(")[0][-60:]
    if "daso" in name or any(k + "<" in name or k + "(" in name for k in OURS):
        base = name.split("(daso::")[0] if "(daso::" in name else name.split("(")[0]
        return "libdaso::" + base.split("::")[-1]
    if "nccl" in name.lower():
        return "nccl::" + name.split("(")[0][:60]
    return "other: " + name[:70]


def launches(path, out, about):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        a = agg.setdefault(short(r[ki]), {"launches": 0, "us_total": 0.0})
        a["launches"] += 1
        a["us_total"] += float(r[vi]) / 1e3
    tot = sum(v["us_total"] for v in agg.values())
    for v in agg.values():
        v["us_per_launch"] = v["us_total"] / v["launches"]
        v["share_of_all_launches"] = v["us_total"] / tot
    json.dump({"about": about, "kernels": agg}, open(out, "w"), indent=1)
    return agg


def full(rep, out, about, key=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    ls = [{k: r[hdr.index(k)] for k in KEYS if k in hdr} for r in rows[2:]]
    tr = [(float(l["dram__bytes_read.sum"]) + float(l["dram__bytes_write.sum"])) * 1e6 for l in ls]
    d = {"about": about, "units": {k: rows[1][hdr.index(k)] for k in KEYS if k in hdr}, "launches": ls,
         "dram_bytes_per_launch_mean": sum(tr) / len(tr)}
    json.dump(d, open(out, "w"), indent=1)
    if key:
        p = "profiles/ncu_traffic.json"
        try:
            t = json.load(open(p))
        except Exception:
            t = {}
        t[key] = {"dram_bytes_per_launch": d["dram_bytes_per_launch_mean"], "source": out}
        json.dump(t, open(p, "w"), indent=1)
    return d


if __name__ == "__main__":
    kind = sys.argv[1]
    if kind == "launches":
        print(json.dumps(launches(*sys.argv[2:5]), indent=1))
    else:
        d = full(*sys.argv[2:6])
        print(d["dram_bytes_per_launch_mean"], len(d["launches"]))
