#!/usr/bin/env python
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/<round>_*.{md,json}.

  python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.md
  python scripts/ncu_summary.py full gpurun_out/prof_conv.ncu-rep profiles/r01_conv.md [--traffic-key conv_fprop]
"""
import csv
import collections
import io
import json
import os
import re
import subprocess
import sys

NCU = os.environ.get("NCU", "ncu")


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"void |xp::|\(anonymous namespace\)::", "", name)
    return name[:90]


def launches(csv_path, out_md):
    rows = []
    with open(csv_path) as f:
        txt = f.read()
    i = txt.find('"ID"')
    rd = csv.DictReader(io.StringIO(txt[i:]))
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        rows.append((short(r["Kernel Name"]), ns))
    tot = sum(ns for _, ns in rows)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, ns in rows:
        agg[n][0] += 1
        agg[n][1] += ns
    lines = ["# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)", "",
             "%d launches, %.3f ms total" % (len(rows), tot / 1e6), "",
             "| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for n, (cnt, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append("| %s | %d | %.1f | %.1f%% | %.2f |" % (n, cnt, ns / 1e3, 100 * ns / tot, ns / 1e3 / cnt))
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    return {n: {"launches": c, "us": ns / 1e3, "share": ns / tot} for n, (c, ns) in agg.items()}


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__warps_active.avg.per_cycle_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__block_size"]


def full(rep, out_md, traffic_key=None):
    if rep.endswith(".csv"):  # a raw-page CSV exported on the box (ncu -i ... --page raw --csv)
        out = open(rep).read()
    else:
        out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rd = list(csv.reader(io.StringIO(out)))
    if len(rd) < 3:
        raise SystemExit("no data in " + rep)
    hdr, units = rd[0], rd[1]
    res = []
    for row in rd[2:]:
        d = dict(zip(hdr, row))
        item = {"kernel": short(d.get("Kernel Name", "?"))}
        stalls = []
        for k in hdr:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(d[k].replace(",", "")), k))
                except ValueError:
                    pass
        for v, k in sorted(stalls, reverse=True)[:6]:  # the dominant warp stall reasons
            item[k] = "%.2f cycles per issued instruction" % v
        for k in hdr:
            if k in WANT or ("tensor" in k and "pct" in k and ".avg." in k):
                if k not in WANT and d[k].strip() in ("0", "0.000000", ""):
                    continue  # drop the all-zero tensor sub-pipe rows (noise)
                item[k] = d[k] + " " + units[hdr.index(k)]
        res.append(item)
    lines = ["# ncu --set full summary: %s" % os.path.basename(rep), ""]
    for it in res:
        lines.append("## " + it["kernel"])
        for k, v in it.items():
            if k != "kernel":
                lines.append("- %s: %s" % (k, v))
        lines.append("")
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic_key:
        def num(s):
            v, u = s.split(" ", 1) if " " in s else (s, "")
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u.strip(), 1)
        tb = [num(it["dram__bytes_read.sum"]) + num(it["dram__bytes_write.sum"]) for it in res
              if "dram__bytes_read.sum" in it]
        if tb:
            path = os.path.join(os.path.dirname(out_md), "traffic.json")
            cur = json.load(open(path)) if os.path.exists(path) else {}
            cur[traffic_key] = sum(tb) / len(tb)
            json.dump(cur, open(path, "w"), indent=1)
    return res


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
        full(sys.argv[2], sys.argv[3], key)
