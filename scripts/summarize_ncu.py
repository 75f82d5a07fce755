"""Summarise ncu captures (gpurun_out/*.ncu-rep, launch lists) into small
committed JSON files under profiles/.

    python scripts/summarize_ncu.py <name> <report.ncu-rep> [config_key algorithmic_bytes]
    python scripts/summarize_ncu.py --launches <launches.csv> <name>
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "dram__cycles_elapsed.avg.per_second",
           "sm__cycles_elapsed.avg.per_second"]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return v


def summarize(name, rep, key=None, alg_bytes=None):
    rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"report": os.path.basename(rep), "kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None,
           "metrics": {}, "stalls_top": {}, "sass_mix_top": {}}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            out["metrics"][m] = {"value": to_num(vals[i]), "unit": units[i]}
    st = []
    for i, h in enumerate(hdr):
        if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
            v = to_num(vals[i])
            if isinstance(v, float):
                st.append((v, h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    tot = sum(v for v, _ in st) or 1
    out["stalls_top"] = {h: round(100 * v / tot, 1) for v, h in sorted(st, reverse=True)[:8]}
    sass = ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"])
    if len(sass) > 2:
        h = sass[1]
        iS, iE = h.index("Source"), h.index("Instructions Executed")
        mix = collections.Counter()
        for r in sass[2:]:
            if len(r) != len(h):
                continue
            m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS].strip())
            mix[m.group(2) if m else "?"] += int(r[iE] or 0)
        t = sum(mix.values()) or 1
        out["sass_mix_top"] = {k: round(100 * v / t, 1) for k, v in mix.most_common(14)}
        out["sass_mnemonics_present"] = sorted({k for k in mix if k.startswith(("UBLKCP", "SYNCS", "UTMA", "LDS", "STG", "LDG"))})
    rd = out["metrics"].get("dram__bytes_read.sum", {}).get("value")
    wr = out["metrics"].get("dram__bytes_write.sum", {}).get("value")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    urd = scale.get(out["metrics"].get("dram__bytes_read.sum", {}).get("unit", ""), 1)
    uwr = scale.get(out["metrics"].get("dram__bytes_write.sum", {}).get("unit", ""), 1)
    if rd is not None and wr is not None:
        out["dram_bytes_per_launch"] = rd * urd + wr * uwr
        if alg_bytes:
            out["algorithmic_bytes_per_launch"] = alg_bytes
            out["traffic_over_algorithmic"] = out["dram_bytes_per_launch"] / alg_bytes
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    if key:
        tp = os.path.join(PROF, "relax_traffic.json")
        d = json.load(open(tp)) if os.path.exists(tp) else {}
        d[key] = {"dram_bytes_per_launch": out["dram_bytes_per_launch"], "source": f"profiles/{name}.json",
                  "kernel": out["kernel"]}
        json.dump(d, open(tp, "w"), indent=1)
    print(json.dumps(out, indent=1)[:3000])


def launches(path, name):
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if "Kernel Name" in r][0]
    data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r != hdr]
    agg = collections.OrderedDict()
    for d in data:
        k = re.sub(r"\(.*", "", d["Kernel Name"])[:80]
        agg.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = {"source": os.path.basename(path), "note": "ncu --metrics gpu__time_duration.sum --clock-control none "
           "(cold-cache, serialised: compare shares)", "kernels": {}}
    for k, v in agg.items():
        out["kernels"][k] = {"launches": len(v), "mean_ns": sum(v) / len(v), "share_of_device_time": sum(v) / tot}
    with open(os.path.join(PROF, f"{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        summarize(sys.argv[1], sys.argv[2], *(sys.argv[3:4] or [None]),
                  *(float(sys.argv[4]),) if len(sys.argv) > 4 else ())
