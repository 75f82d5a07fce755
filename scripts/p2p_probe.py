"""One local and one push-mode (self-exchange) solve of a slab of BASELINE
config 3 (16384 x 16384/P rows), for a kernel launch list under ncu:
    ncu --metrics gpu__time_duration.sum python scripts/p2p_probe.py [P] [N]"""
import os
import sys

os.environ["PROTOX_NCCL_SELF_EXCHANGE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
N = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n0, n1 = 16384, 16384 // p
h = 1.0 / n0
lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (256, 256), 1, P.PX_BC_PERIODIC, 1)
a, b, r = lay.alloc(0), lay.alloc(0), lay.alloc(0)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
P.init_field(lay, 0, lay.patch(0, r), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
prm = P.relax_params(h, h * h / 8)
pa, pb, pr = lay.patch(0, a), lay.patch(0, b), lay.patch(0, r)
P.solve(lay, None, 0, prm, N, 1, pa, pb, pr, use_graph=False, stream=s)
comm = P.Comm(None, 1, 0, torch.cuda.current_device())
P.comm_p2p_import(comm, lay, [P.comm_p2p_export(comm, lay, 0, pa, pb)])
P.solve(lay, comm, 0, prm, N, 1, pa, pb, pr, use_graph=False, stream=s)
torch.cuda.synchronize()
comm.close()
print("ok")
