"""Summarise an ncu SASS source-page export (prof_*_sass.csv.gz written by
scripts/prof_tb.sh): stall mix, op mix of the hottest straight-line body."""
import collections
import csv
import gzip
import re
import sys

path = sys.argv[1]
raw = sys.argv[2] if len(sys.argv) > 2 else None
if raw:
    rows = list(csv.reader(open(raw)))
    hdr = rows[0]
    d = dict(zip(hdr, rows[2]))
    st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k].replace(',', ''))) for k in hdr
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and d[k].replace(',', '').replace('.', '').isdigit()]
    st.sort(key=lambda x: -x[1])
    tot = sum(v for _, v in st)
    print("duration_ms", d.get("gpu__time_duration.sum"), "inst", d.get("smsp__inst_executed.sum"),
          "issue%", d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
          "dram%", d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"))
    print("stalls", [(k, round(100 * v / tot, 1)) for k, v in st[:10]])
f = gzip.open(path, "rt")
r = csv.reader(f)
next(r)
hdr = next(r)
ia, isrc, ismp = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
rows = [x for x in r if len(x) > ia]
cnt = [int(x[ia]) for x in rows]
tot = sum(cnt)
byc = collections.Counter()
for c in cnt:
    byc[c] += c
c0, t0 = byc.most_common(1)[0]
body = [x for x in rows if int(x[ia]) == c0]
print(f"total inst {tot}; hottest body: {len(body)} instructions x {c0} = {100 * t0 / tot:.1f}%")
ops, smp = collections.Counter(), collections.Counter()
for x in body:
    op = re.sub(r"^@!?U?P\w+\s+", "", x[isrc].strip()).split(" ")[0]
    ops[op] += 1
    smp[op] += int(x[ismp])
for k, v in ops.most_common(25):
    print(f"  {k:26s} {v:4d}  samples {smp[k]}")
