"""One-GPU A/B of the multi-GPU solve paths at 16384² (PROTOX_NCCL_SELF_EXCHANGE=1:
the one-rank periodic layout exchanges its ghost rows with itself):
  local  -- no communicator (fused wrap images)
  nccl   -- boundary rows, grouped ncclSend/ncclRecv on the comm stream, interior overlapped
  p2p    -- boundary-row kernels push into the neighbour's ghost rows over peer memory
Prints ms per sweep of a 100-sweep graph-replayed solve, norms every sweep."""
import json
import os
import sys

os.environ["PROTOX_NCCL_SELF_EXCHANGE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

n, N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384, 100
lay = P.Layout(P.box(0, 0, n - 1, n - 1), (256, 256), 1, P.PX_BC_PERIODIC, 1)
a, b, r = lay.alloc(0), lay.alloc(0), lay.alloc(0)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
P.init_field(lay, 0, lay.patch(0, r), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
prm = P.relax_params(1.0 / n, (1.0 / n) ** 2 / 8)
pa, pb, pr = lay.patch(0, a), lay.patch(0, b), lay.patch(0, r)
out = {"n": n}
for mode in ("local", "nccl", "p2p"):
    comm = None
    if mode != "local":
        comm = P.Comm(P.comm_unique_id(), 1, 0, torch.cuda.current_device())
        if mode == "p2p":
            P.comm_enable_p2p(comm, lay, 0, pa, pb)
    run = lambda: P.solve(lay, comm, 0, prm, N, 1, pa, pb, pr, use_graph=True, stream=s)
    run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5):
        run()
    e1.record(s)
    s.synchronize()
    out[mode + "_ms_per_sweep"] = e0.elapsed_time(e1) / (5 * N)
    if comm:
        comm.close()
print(json.dumps(out))
