"""Re-run the paper's CPU experiment (figure `runtime`
P:320-325) on this host: Proto (unfused) vs ProtoX (fused) run time, 4 x 4
periodic boxes of 64², 128², 256² cells, 100 Jacobi iterations, 1 thread and
an OpenMP team.  Context for the GPU numbers; the
paper reports "up to 2x" on a 2.3 GHz quad-core i7.

    python scripts/cpu_fusion_ratio.py [out.json]
"""
import json
import os
import platform
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hostref  # noqa: E402
from paper_2307_07931_b200 import inputs  # noqa: E402


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else None
    nproc = os.cpu_count() or 1
    teams = sorted({1, min(4, nproc), nproc})
    rows = []
    for box in (64, 128, 256):
        n = 4 * box
        h = 1.0 / n
        lam = h * h / 8
        rho = inputs.hash_field(n, n)
        for t in teams:
            best = {}
            for variant in (0, 1):
                times = []
                for _ in range(3):
                    _, sec, _ = hostref.run(variant, box, 4, 100, h, lam, rho, t)
                    times.append(sec)
                best[variant] = min(times)
            rows.append({"box": box, "domain": n, "threads": t, "proto_unfused_s": best[0],
                         "protox_fused_s": best[1], "speedup_fused_over_unfused": best[0] / best[1],
                         "fused_Gcell_updates_per_s": n * n * 100 / best[1] / 1e9})
            print(json.dumps(rows[-1]), flush=True)
    res = {"what": "PAPER.md:212 / figure `runtime` re-run on this host: Proto (unfused: exchange, laplace pass, "
                   "update pass, exchange + residual pass per iteration) vs ProtoX (one fused loop per box, "
                   "Fig. ProtoX), 4x4 periodic boxes, 100 iterations, same data structures and flags "
                   "(g++ -O3 -march=native -fopenmp -ffp-contract=off), best of 3",
           "paper": "up to 2x on a 2.3 GHz quad-core Intel i7 (P:212, P:323)",
           "host": {"cpu": cpu_model(), "nproc": nproc}, "rows": rows}
    if out_path:
        with open(out_path, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
