"""A/B timing of the fused relax kernel variants on one GPU (CUDA events on
the launching stream).  Select the variant with PROTOX_KERNEL=ldg (register
streaming, LDG.128) or unset (TMA bulk-copy pipeline when eligible).

    PROTOX_KERNEL=ldg python scripts/ab_relax.py --n 16384
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--stencil", type=int, default=0)
ap.add_argument("--norms", type=int, default=1)
args = ap.parse_args()
n = args.n
lay = P.Layout(P.box(0, 0, n - 1, n - 1), (min(256, n), min(256, n)), 1, P.PX_BC_PERIODIC, 1)
li = lay.local(0)
a, b, r = lay.alloc(0), lay.alloc(0), lay.alloc(0)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
P.init_field(lay, 0, lay.patch(0, r), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
P.init_field(lay, 0, lay.patch(0, a), P.PX_FIELD_HASH, 7, stream=s)
P.fill_ghosts(lay, 0, lay.patch(0, a), stream=s)
nb = P.norm_buffer(li.owned)
s.wait_stream(torch.cuda.current_stream())
prm = P.relax_params(1.0 / n, (1.0 / n) ** 2 / 8, args.stencil)
pa, pb, pr = lay.patch(0, a), lay.patch(0, b), lay.patch(0, r)
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
for i in range(args.reps):
    evs[i][0].record(s)
    P.relax_step(prm, pa if i % 2 == 0 else pb, pb if i % 2 == 0 else pa, pr, li.owned,
                 nb if args.norms else None, stream=s)
    evs[i][1].record(s)
s.synchronize()
ts = [x.elapsed_time(y) for x, y in evs[3:]]
ms = statistics.median(ts)
gbs = 24 * n * n / (ms * 1e-3) / 1e9
print(json.dumps({"kernel": os.environ.get("PROTOX_KERNEL", "bulk"), "n": n, "stencil": args.stencil,
                  "ms_median": ms, "ms_min": min(ts), "GBps": gbs, "Gcell_s": n * n / (ms * 1e-3) / 1e9,
                  "norm": nb[:2].tolist()}))

if os.environ.get("PROTOX_CEILING"):
    # K12 ceiling on the same byte count: 2 reads + 1 write of n*n doubles
    m = n * n
    x = torch.rand(m, dtype=torch.float64, device="cuda")
    y = torch.rand(m, dtype=torch.float64, device="cuda")
    z = torch.empty(m, dtype=torch.float64, device="cuda")
    for variant, nbytes in ((0, 24 * m), (1, 16 * m)):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for e0, e1 in evs:
            e0.record(s)
            P.stream_ceiling(x, y, z, variant, stream=s)
            e1.record(s)
        s.synchronize()
        ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs[3:])
        print(json.dumps({"kernel": "ceiling_triad" if variant == 0 else "ceiling_copy", "n": n,
                          "ms_median": ms, "GBps": nbytes / (ms * 1e-3) / 1e9}))
    # torch's own copy for reference (MEASURED_PEAKS method, fp64)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    with torch.cuda.stream(s):
        for e0, e1 in evs:
            e0.record(s)
            z.copy_(x)
            e1.record(s)
    s.synchronize()
    ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs[3:])
    print(json.dumps({"kernel": "torch_copy", "n": n, "ms_median": ms, "GBps": 16 * m / (ms * 1e-3) / 1e9}))
