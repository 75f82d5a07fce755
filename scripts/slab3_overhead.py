"""Per-sweep overhead of the 3D z-slab solve paths at the P-rank slab shapes
of the 512³ extension (512 x 512 x 512/P planes, periodic, 7-point), on ONE
GPU: local (one rank, ghost fill only) vs NCCL self-exchange (the rank sends
its boundary planes to itself with the library's grouped send/recv).  ms per
sweep of a 100-sweep graph-replayed solve with norms every sweep."""
import json
import os
import sys

os.environ["PROTOX_NCCL_SELF_EXCHANGE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

N = 100
for p in [int(a) for a in sys.argv[1:]] or [8, 4, 1]:
    n = (512, 512, 512 // p)
    g = P.Grid3(n, 1)
    a, b, r = g.alloc(), g.alloc(), g.alloc()
    P.init_field3(g, r, 1, inputs.DEFAULT_SEED)
    h = 1.0 / 512
    prm = P.relax_params(h, h * h / 12, P.PX_LAPLACE_7PT_3D)
    out = {"P": p, "slab": list(n)}
    for mode in ("local", "nccl"):
        comm = P.Comm(P.comm_unique_id(), 1, 0, torch.cuda.current_device()) if mode == "nccl" else None
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        run = (lambda: P.solve3(g, P.PX_BC_PERIODIC, prm, N, 1, a, b, r, use_graph=True, stream=s)) if comm is None \
            else (lambda: P.solve3_comm(comm, g, P.PX_BC_PERIODIC, prm, N, 1, a, b, r, use_graph=True, stream=s))
        run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            run()
        e1.record(s)
        s.synchronize()
        out[mode + "_ms_per_sweep"] = e0.elapsed_time(e1) / (3 * N)
        if comm:
            P.release3()
            comm.close()
    out["nccl_over_local"] = out["nccl_ms_per_sweep"] / out["local_ms_per_sweep"] - 1
    print(json.dumps(out), flush=True)
    del a, b, r
    torch.cuda.empty_cache()
