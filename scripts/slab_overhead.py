"""Per-sweep overhead of the multi-GPU solve paths at the slab shapes of
BASELINE config 3 split over P ranks (16384 x 16384/P per rank), on ONE GPU.

For each slab shape (n0 = 16384 columns, n1 = 16384/P rows, periodic):
  kernel  -- one px_relax_step over the slab (the sweep kernel alone), CUDA
             events on its stream, mean of 20 after 3 warm-ups
  local   -- px_solve without a communicator (fused wrap images), 100 sweeps,
             norms every sweep, graph replay
  nccl    -- PROTOX_NCCL_SELF_EXCHANGE=1: the one-rank layout sends its ghost
             rows to itself with the grouped NCCL send/recv of the halo plan on
             the comm stream, boundary rows first, interior overlapped
  p2p     -- the same with the peer-memory push (px_comm_enable_p2p)
Prints one JSON object: ms per sweep of each path and the overhead over the
kernel alone (the fixed per-sweep cost that limits strong-scaling efficiency).

    python scripts/slab_overhead.py [P ...]     (default 8 4 2 1)
"""
import json
import os
import sys

os.environ["PROTOX_NCCL_SELF_EXCHANGE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

N = 100
ps = [int(a) for a in sys.argv[1:]] or [8, 4, 2, 1]
n0 = 16384
rows = []
for p in ps:
    n1 = 16384 // p
    h = 1.0 / n0
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (256, 256), 1, P.PX_BC_PERIODIC, 1)
    li = lay.local(0)
    a, b, r = lay.alloc(0), lay.alloc(0), lay.alloc(0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    P.init_field(lay, 0, lay.patch(0, r), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
    prm = P.relax_params(h, h * h / 8)
    pa, pb, pr = lay.patch(0, a), lay.patch(0, b), lay.patch(0, r)
    out = {"P": p, "slab": [n0, n1], "lib": os.path.basename(P.LIB_PATH)}
    # the sweep kernel alone
    nb = P.norm_buffer(li.owned)
    s.wait_stream(torch.cuda.current_stream())
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(23)]
    for i, (e0, e1) in enumerate(evs):
        src, dst = (pa, pb) if i % 2 == 0 else (pb, pa)
        e0.record(s)
        P.relax_step(prm, src, dst, pr, li.owned, nb, stream=s)
        e1.record(s)
    s.synchronize()
    out["kernel_ms"] = sum(e0.elapsed_time(e1) for e0, e1 in evs[3:]) / 20
    for mode in os.environ.get("SLAB_MODES", "local,nccl,p2p").split(","):
        comm = None
        if mode != "local":
            comm = P.Comm(P.comm_unique_id(), 1, 0, torch.cuda.current_device())
            if mode == "p2p":
                P.comm_enable_p2p(comm, lay, 0, pa, pb)
        run = lambda: P.solve(lay, comm, 0, prm, N, 1, pa, pb, pr, use_graph=True, stream=s)
        run()
        out[mode + "_kernels"] = P.last_solve_kernels()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5):
            run()
        e1.record(s)
        s.synchronize()
        ms = e0.elapsed_time(e1) / (5 * N)
        out[mode + "_ms_per_sweep"] = ms
        out[mode + "_overhead_frac"] = ms / out["kernel_ms"] - 1
        if comm:
            comm.close()
    P.release_cached()
    del a, b, r
    torch.cuda.empty_cache()
    rows.append(out)
    print(json.dumps(out), flush=True)
