#!/usr/bin/env python
"""bench.py -- fp64 Gcell-updates/s of the fused relax sweep (BASELINE.json metric).

Default workload (N=1): BASELINE config 3, a 16384x16384 fp64 periodic 2D
Poisson problem, 5-point Laplacian, slab layout of 256x256 boxes, ρ = the
seeded counter-hash field (synthetic, generated on the device), φ0 = 0,
h = 2^-14, λ = h²/8.  One STEP = one px_solve of 100 Jacobi sweeps (the
paper's fixed 100 iterations) with the residual max/L2 norm recorded
every sweep, replayed from a CUDA graph; the multi-GPU run splits the same
16384² domain into slabs over N ranks (strong scaling) with a per-sweep
NCCL ghost exchange and the residual all-reduce.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3|C2|C1|C4|C5|C3D]
    python bench.py --impl reference ...   # the CPU oracle on a bounded sample

Prints ONE JSON line on rank 0.  Inputs (3 x 2.15 GB) exceed the 126 MB L2,
so no L2 flush is needed between steps (config.l2 says so).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 Gcell-updates/s of fused relax sweep at 1/2/4/8 B200; % HBM roofline"
UNIT = "Gcell-updates/s"
BYTES_PER_CELL_UPDATE = 24  # read φ 8 + read ρ 8 + write φ' 8

# the whole-solve kernels of the small configs (named by px_last_solve_kernels)
SOLVE_KERNELS = {
    "k_resident_reg": "iterate in registers, rows resident on chip across all sweeps, LL row mailbox in L2 "
                      "between neighbouring CTAs, one launch",
    "k_resident_reg2": "k_resident_reg with two sweeps per mailbox hop",
    "k_resident": "iterate resident in shared memory, LL row mailbox, one launch",
    "k_boxw": "whole box in registers on one CTA, one warp per row group, one launch",
    "k_cluster_box": "whole solve on an 8-CTA cluster, DSMEM halos, one launch",
    "k_box1": "whole box on one CTA of 1024 threads, one launch",
    "k_smallbox": "whole box in shared memory on one CTA, one launch",
}

CONFIGS = {
    "C3": dict(n=16384, box=256, bc=0, stencil=0, sweeps=100, norm_every=1, rho="hash",
               desc="BASELINE config 3: 2D Poisson 16384x16384 fp64, periodic, 5-point, "
                    "slab-decomposed, per-sweep ghost exchange and residual all-reduce"),
    "C4": dict(n=32768, box=256, bc=0, stencil=0, sweeps=100, norm_every=4, rho="hash", ghost=4, tk=4,
               desc="BASELINE config 4: 2D Poisson 32768x32768 fp64, periodic, 5-point, 256x256-box "
                    "DisjointBoxLayout, temporal blocking k=4 sweeps per halo exchange (norm per exchange)"),
    "C2": dict(n=1024, box=1024, bc=0, stencil=0, sweeps=1000, norm_every=10, rho="hash",
               solve_kernel=True,
               desc="BASELINE config 2: 2D Poisson 1024x1024 single box, 1000 sweeps, "
                    "max-norm every 10 (L2-resident)"),
    "C1": dict(n=64, box=64, bc=1, stencil=0, sweeps=100, norm_every=1, rho="sine",
               solve_kernel=True,
               desc="BASELINE config 1: 64x64 box + 1 ghost layer, Dirichlet, 100 sweeps"),
    "C5": dict(n=8192, box=256, bc=1, stencil=1, sweeps=100, norm_every=1, rho="sine",
               desc="BASELINE config 5: 8192x8192 Mehrstellen 9-point, Dirichlet-CC"),
    "C3D": dict(n=512, box=512, bc=0, stencil=2, sweeps=100, norm_every=1, rho="hash", dims=3,
                desc="3D extension (SURVEY 8(f) rank 3, not a BASELINE config): 3D Poisson 512^3 fp64, "
                     "periodic, 7-point, norms every sweep"),
    "C3D27": dict(n=512, box=512, bc=1, stencil=3, sweeps=100, norm_every=1, rho="hash", dims=3,
                  desc="3D extension (SURVEY 8(f) rank 3): 3D Poisson 512^3 fp64, Dirichlet-CC, 27-point "
                       "compact Mehrstellen with the corrected right-hand side, norms every sweep"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--halo", default="p2p", choices=["nccl", "p2p"],
                    help="multi-GPU ghost exchange: the fused peer-memory push inside the relax kernel "
                         "(px_comm_enable_p2p, default; self-checked against NCCL at start-up, NCCL if it "
                         "fails) or NCCL grouped send/recv on a comm stream")
    ap.add_argument("--no-halo-proxy", action="store_true",
                    help="N = 1: skip the one-GPU halo-path measurement at the 8-rank slab shape")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(config):
    """Per-launch DRAM bytes of the relax kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "relax_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(config)
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


def k12_ceiling(P, torch, dev, elems: int, stream) -> float:
    """K12: the box's own 2-read/1-write fp64 streaming ceiling
    (c = a + b over arrays of the sweep's size, px_stream_ceiling), GB/s,
    CUDA events on the launching stream, median of 7 after 2 warm-ups."""
    a = torch.empty(elems, dtype=torch.float64, device=dev).fill_(1.0)
    b = torch.empty_like(a).fill_(2.0)
    c = torch.empty_like(a)
    stream.wait_stream(torch.cuda.current_stream(dev))
    ms = []
    for i in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        P.stream_ceiling(a, b, c, 0, stream=stream)
        e1.record(stream)
        stream.synchronize()
        if i >= 2:
            ms.append(e0.elapsed_time(e1))
    del a, b, c
    return 24 * elems / (statistics.median(ms) * 1e-3) / 1e9


def roofline_extras(roof: dict, cells_per_launch: int, ceiling_gbps: float | None):
    """The three denominators of SURVEY §8(d) and the effective bytes per cell:
    the 8 TB/s spec, the measured copy bandwidth (MEASURED_PEAKS.json, = the
    line's `peak`), the live K12 streaming ceiling."""
    ach = roof["achieved"]
    roof["frac_vs_spec_8000"] = ach / 8000.0
    if ceiling_gbps:
        roof["k12_ceiling_GBps"] = ceiling_gbps
        roof["frac_vs_k12_ceiling"] = ach / ceiling_gbps
    if roof.get("traffic"):
        roof["effective_bytes_per_cell_per_launch"] = roof["traffic"] / cells_per_launch
    return roof


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw,power.limit")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        pw = [v for v in (num(r[7]) for r in self.rows if len(r) > 8) if v is not None]
        pl = [v for v in (num(r[8]) for r in self.rows if len(r) > 8) if v is not None]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                # board power under load against its limit: sw_power_cap explains a
                # compute-heavier kernel (C4) running below max clocks
                "power_w": statistics.median(pw) if pw else None, "power_limit_w": max(pl) if pl else None}


# ----------------------------------------------------------------- oracle arm
def oracle_sample(cfg, n_sample: int, sweeps: int):
    """Run the CPU oracle (test infrastructure, allowed here for cpu_baseline /
    --impl reference only) on a bounded sample of the workload."""
    import numpy as np

    import oracle
    from paper_2307_07931_b200 import inputs
    n = n_sample
    h = 1.0 / n
    bc = {0: oracle.BC_PERIODIC, 1: oracle.BC_DIRICHLET_CC}[cfg["bc"]]
    lam = h * h / 8
    box = min(cfg["box"], n)
    p = oracle.Problem(n, n, h, lam, b0=box, b1=box, bc=bc, stencil=cfg["stencil"],
                       nsweeps=sweeps, norm_every=cfg["norm_every"])
    rho = inputs.hash_field(n, n) if cfg["rho"] == "hash" else inputs.sine_field(n, n)
    rho_g = oracle.ghosted(p, rho)
    phi_g = np.zeros_like(rho_g)
    t0 = time.perf_counter()
    oracle.solve(p, phi_g, rho_g)
    dt = time.perf_counter() - t0
    return n * n * sweeps / dt / 1e9, dt


def oracle_sample3(cfg, n_sample: int, sweeps: int):
    """The 3D oracle on an n_sample³ sample of the same recipe."""
    import numpy as np

    import oracle
    from paper_2307_07931_b200 import inputs
    n = n_sample
    h = 1.0 / n
    p = oracle.Problem3((n, n, n), h, h * h / 12, bc=oracle.BC_PERIODIC if cfg["bc"] == 0 else oracle.BC_DIRICHLET_CC,
                        nsweeps=sweeps, norm_every=cfg["norm_every"], stencil=0 if cfg["stencil"] == 2 else 1,
                        rhs_correction=cfg["stencil"] == 3)
    rho_g = oracle.ghosted3(p, inputs.hash_field3(n, n, n))
    phi_g = np.zeros_like(rho_g)
    t0 = time.perf_counter()
    oracle.solve3(p, phi_g, rho_g)
    dt = time.perf_counter() - t0
    return n ** 3 * sweeps / dt / 1e9, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    if cfg.get("dims") == 3:
        n_s, sweeps = 128, 20
        rates, times = [], []
        for i in range(args.warmup + args.steps):
            r, dt = oracle_sample3(cfg, n_s, sweeps)
            if i >= args.warmup:
                times.append(dt)
        total = n_s ** 3 * sweeps * args.steps / sum(times) / 1e9
        sample = f"3D oracle (single-threaded C++, unfused Proto order) on {n_s}^3, {sweeps} sweeps per step"
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": total, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg["desc"], "sample": sample},
            "cpu_baseline": {"value": total, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": total, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return 0
    n_s = min(cfg["n"], 2048)
    sweeps = 10 if cfg["n"] > 2048 else cfg["sweeps"]
    for _ in range(args.warmup):
        oracle_sample(cfg, n_s, sweeps)
    rates, times = [], []
    for _ in range(args.steps):
        r, dt = oracle_sample(cfg, n_s, sweeps)
        rates.append(r)
        times.append(dt)
    total = n_s * n_s * sweeps * args.steps / sum(times) / 1e9
    sample = f"oracle (single-threaded C++, unfused Proto order) on {n_s}x{n_s} of the same recipe, {sweeps} sweeps per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": total, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": cfg["desc"], "sample": sample},
        "cpu_baseline": {"value": total, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": total, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------- native arm
def run_native3d(args):
    """C3D / C3D27: the 3D relaxation (px3_solve).  N > 1: the n³ domain in
    z-slabs over the ranks (px3_solve_comm: z ghost planes over NCCL, norms
    all-reduced at the end) -- strong scaling."""
    import torch
    import torch.distributed as dist

    from paper_2307_07931_b200 import inputs
    from paper_2307_07931_b200 import protox as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PROTOX_BENCH_SHARED_GPU=1 (tests only): every rank on cuda:0, gloo process
    # group, no NCCL communicator -- exercises the N > 1 code path (push halo,
    # halo metrics, max-over-ranks timing, e2e) on a one-GPU box
    shared = world > 1 and os.environ.get("PROTOX_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfg = CONFIGS[args.config]
    if shared and (cfg.get("tk", 1) > 1 or cfg["stencil"] == 1 or args.halo != "p2p"):
        raise SystemExit("PROTOX_BENCH_SHARED_GPU: k = 1, 5-point, --halo p2p only")
    n, S, E = cfg["n"], cfg["sweeps"], cfg["norm_every"]
    h = 1.0 / n
    lam = h * h / 12  # λ = h²/(4D), D = 3
    comm = None
    nzl = n
    if world > 1 and cfg["stencil"] != P.PX_LAPLACE_7PT_3D:
        raise SystemExit("C3D27 runs on one GPU (its corrected right-hand side needs exchanged rho planes)")
    if world > 1:
        z0, z1 = P.slab3(n, world, rank)
        nzl = z1 - z0
        obj = [P.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = P.Comm(obj[0], world, rank, local)
    grid = P.Grid3((n, n, nzl), 1)
    phi, scr, rho = grid.alloc(dev), grid.alloc(dev), grid.alloc(dev)
    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream(dev))
    prm = P.relax_params(h, lam, cfg["stencil"])
    P.init_field3(grid, rho, 1, inputs.DEFAULT_SEED, stream=stream, z0=z0 if world > 1 else 0)
    if cfg["stencil"] == P.PX_MEHRSTELLEN_27PT_3D:  # f = ρ + S7(ρ)/12 (ρ ghosts by the BC rule)
        P.fill_ghosts3(grid, cfg["bc"], rho, stream=stream)
        f = grid.alloc(dev)
        stream.wait_stream(torch.cuda.current_stream(dev))
        P.mehrstellen_rhs3(grid, rho, f, stream=stream)
        rho = f
    stream.synchronize()
    bufs = [phi, scr]

    def solve_any(a, b, r_):
        if comm is not None:
            return P.solve3_comm(comm, grid, cfg["bc"], prm, S, E, a, b, r_, use_graph=True, stream=stream)
        return P.solve3(grid, cfg["bc"], prm, S, E, a, b, r_, use_graph=True, stream=stream)

    def step():
        r = solve_any(bufs[0], bufs[1], rho)
        if r.in_scratch:
            bufs.reverse()
            tens.reverse()
        return r

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        res = step()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = P.kernel_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        res = step()
    ev1.record(stream)
    barrier()
    launches = P.kernel_launch_count() - launches0
    clk = clocks.stop()
    t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    value = n ** 3 * S * args.steps / (t_ms * 1e-3) / 1e9

    # roofline of k3_relax (px3_relax_step, same launch geometry), CUDA events on its stream
    nb = P.norm_buffer3(dev)
    stream.wait_stream(torch.cuda.current_stream(dev))
    reps = 20
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for i in range(reps):
        src, dst = (bufs[0], bufs[1]) if i % 2 == 0 else (bufs[1], bufs[0])
        P.fill_ghosts3(grid, cfg["bc"], src, stream=stream)
        evs[i][0].record(stream)
        P.relax_step3(prm, grid, src, dst, rho, nb, stream=stream)
        evs[i][1].record(stream)
    stream.synchronize()
    k_ms = statistics.mean(a.elapsed_time(b) for a, b in evs[2:])
    alg = BYTES_PER_CELL_UPDATE * n * n * nzl
    peak, peak_src = load_peaks()
    roofline = {"bound": "hbm", "achieved": alg / (k_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                "frac": alg / (k_ms * 1e-3) / 1e9 / peak, "traffic": load_traffic(args.config) if world == 1 else None,
                "kernel": "k3_relax<RELAX,%s> (3D, TMA tensor tiles marching in z)"
                          % ("7pt" if cfg["stencil"] == P.PX_LAPLACE_7PT_3D else "27pt"), "kernel_ms": k_ms,
                "algorithmic_bytes_per_launch": alg, "peak_source": peak_src,
                "whole_step_GBps": BYTES_PER_CELL_UPDATE * value / world}
    roofline_extras(roofline, n * n * nzl, k12_ceiling(P, torch, dev, n * n * nzl, stream))

    # e2e: pinned host ρ -> device, solve from φ0 = 0, φ^N back to pinned host, every step.
    # N = 1: px3_solve_host_batch (one problem per step, copies of neighbouring
    # steps overlapped with the solve); N > 1: torch copies around px3_solve_comm.
    e2e = None
    if not args.no_e2e:
        h_rho = grid.view(rho).cpu().pin_memory()
        h_outs = [torch.empty_like(h_rho).pin_memory() for _ in range(2)]
        if world == 1:
            def e2e_run(k):
                P.solve3_host_batch((n, n, nzl), 1, cfg["bc"], prm, S, E, [h_rho.numpy()] * k,
                                    [h_outs[i % 2].numpy() for i in range(k)], None, use_graph=True,
                                    stream=stream)
        else:
            h_out = h_outs[0]
            d_phi, d_scr, d_rhs = grid.alloc(dev), grid.alloc(dev), grid.alloc(dev)
            stream.wait_stream(torch.cuda.current_stream(dev))

            def e2e_step():
                with torch.cuda.stream(stream):
                    grid.view(d_phi).zero_()
                    grid.view(d_rhs).copy_(h_rho, non_blocking=True)
                r = solve_any(d_phi, d_scr, d_rhs)
                with torch.cuda.stream(stream):
                    h_out.copy_(grid.view(d_scr if r.in_scratch else d_phi), non_blocking=True)
                stream.synchronize()

            def e2e_run(k):
                for _ in range(k):
                    e2e_step()
        e2e_run(3)  # builds the plans / buffers (N = 1: the three pipeline sets)
        barrier()
        ke = max(3, min(args.steps, 6))
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        e2e_run(ke)
        w1.record(stream)
        barrier()
        te = torch.tensor([w0.elapsed_time(w1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        n_norm = (S + E - 1) // E + 1 if E > 0 else 1
        e2e = {"value": n ** 3 * S * ke / (te.item() * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": n * n * nzl * 8, "d2h_bytes_per_step": n * n * nzl * 8 + 16 * n_norm,
               "steps": ke,
               "api": ("px3_solve_host_batch (one problem per step: H2D rho, solve, D2H phi^N + norms; phi0 = 0 "
                       "zero-filled on the device; copies overlap the neighbouring steps' solves)") if world == 1
               else "torch pinned copy of rho + px3_solve_comm (phi0 = 0 zero-filled on the device) + D2H phi^N"}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        r, dt = oracle_sample3(cfg, 160, 20)
        cpu = {"value": r, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"single-threaded C++ 3D oracle, 160^3 of the same recipe, 20 sweeps, {dt:.1f} s"}
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "n": n, "sweeps_per_step": S, "norm_every": E, "ghost": 1,
                       "partition": f"z-slabs x{world}",
                       "rho": cfg["rho"],
                       "h": h, "lambda": lam,
                       "steps_continue": "each step continues from the previous step's iterate",
                       "l2": "inputs (3 x %.2f GB) exceed L2; no flush" % (grid.alloc_elems * 8 / 1e9)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "final_residual_max": float(res.norms[-1, 0]) if len(res.norms) else None}))
    if comm is not None:
        P.release3()
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_native(args):
    import torch
    import torch.distributed as dist

    from paper_2307_07931_b200 import inputs
    from paper_2307_07931_b200 import protox as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PROTOX_BENCH_SHARED_GPU=1 (tests only): every rank on cuda:0, gloo process
    # group, no NCCL communicator -- exercises the N > 1 code path (push halo,
    # halo metrics, max-over-ranks timing, e2e) on a one-GPU box
    shared = world > 1 and os.environ.get("PROTOX_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfg = CONFIGS[args.config]
    if shared and (cfg.get("tk", 1) > 1 or cfg["stencil"] == 1 or args.halo != "p2p"):
        raise SystemExit("PROTOX_BENCH_SHARED_GPU: k = 1, 5-point, --halo p2p only")
    n, S, E = cfg["n"], cfg["sweeps"], cfg["norm_every"]
    h = 1.0 / n
    lam = h * h / 8
    box = cfg["box"]
    ghost, tk = cfg.get("ghost", 1), cfg.get("tk", 1)
    lay = P.Layout(P.box(0, 0, n - 1, n - 1), (box, box), ghost, cfg["bc"], world)
    li = lay.local(rank)
    phi, scr, rho = lay.alloc(rank, dev), lay.alloc(rank, dev), lay.alloc(rank, dev)
    comm = None
    if world > 1 and not shared:
        obj = [P.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = P.Comm(obj[0], world, rank, local)
    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream(dev))  # the zero-fills ran on the current stream
    prm = P.relax_params(h, lam, cfg["stencil"])
    with torch.cuda.stream(stream):
        kind = P.PX_FIELD_HASH if cfg["rho"] == "hash" else P.PX_FIELD_SINE
        P.init_field(lay, rank, lay.patch(rank, rho), kind, inputs.DEFAULT_SEED, 1, 1, stream=stream)
        rhs = rho
        if cfg["stencil"] == 1:
            P.exchange_ghosts(lay, comm, rank, lay.patch(rank, rho), stream=stream)
            rhs = lay.alloc(rank, dev)
            stream.wait_stream(torch.cuda.current_stream(dev))
            P.mehrstellen_rhs(lay.patch(rank, rho), lay.patch(rank, rhs), li.owned, stream=stream)
        if tk > 1:  # temporal blocking advances the halo: ρ needs its ghosts
            P.exchange_ghosts(lay, comm, rank, lay.patch(rank, rhs), stream=stream)
    stream.synchronize()
    pa, pb, pr = lay.patch(rank, phi), lay.patch(rank, scr), lay.patch(rank, rhs)
    halo_mode = "local" if world == 1 else "nccl"
    scomm = comm  # the communicator px_solve uses
    if shared:  # no NCCL to check against: the push path itself is under test
        scomm = P.Comm(None, world, rank, local)
        recs = [None] * world
        dist.all_gather_object(recs, P.comm_p2p_export(scomm, lay, rank, pa, pb))
        P.comm_p2p_import(scomm, lay, recs)
        halo_mode = "p2p (shared-GPU test mode)"
    elif comm is not None and args.halo == "p2p" and tk == 1:
        pcomm, why = p2p_setup(P, torch, dist, lay, rank, world, local, comm, prm, S, pa, pb, pr, phi, stream)
        if pcomm is not None:
            scomm, halo_mode = pcomm, "p2p"
        else:
            halo_mode = f"nccl (p2p refused: {why})"

    bufs = [pa, pb]
    tens = [phi, scr]  # the tensors behind bufs

    # the recorded norms of every step land in device memory (px_solve_async):
    # steps are enqueued back to back, the host reads them after the timed region
    n_ent = ((S + E - 1) // E if E > 0 else 0) + 1
    d_norms = torch.zeros(2 * n_ent, dtype=torch.float64, device=dev)

    def step():
        # each step continues the relaxation from the previous step's iterate (S is even,
        # so with k = 1 the result is back in phi and the registered p2p buffer order holds)
        nw, ins = P.solve_async(lay, scomm, rank, prm, S, E, bufs[0], bufs[1], pr, d_norms, use_graph=True,
                                stream=stream, temporal_k=tk)
        if ins:
            bufs.reverse()
            tens.reverse()
        return nw

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        res = step()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = P.kernel_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        res = step()
    ev1.record(stream)
    barrier()
    launches = P.kernel_launch_count() - launches0
    solve_kernels = P.last_solve_kernels()
    clk = clocks.stop()
    t_ms = max_over_ranks(ev0.elapsed_time(ev1))
    cells = n * n * S * args.steps
    value = cells / (t_ms * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (fused relax sweep, the same
    # k_stream<RELAX> launch geometry over this rank's slab), timed live with
    # CUDA events on the launching stream.
    nb = P.norm_buffer(li.owned, dev)
    stream.wait_stream(torch.cuda.current_stream(dev))
    reps = 20
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    qa, qb = bufs
    for i in range(reps):
        src, dst = (qa, qb) if i % 2 == 0 else (qb, qa)
        if comm is not None or world == 1:  # (shared-GPU test mode: stale ghost rows, timing only)
            P.exchange_ghosts(lay, comm, rank, src, stream=stream)
        evs[i][0].record(stream)
        if tk > 1:
            P.relax_block(prm, tk, src, dst, pr, li.owned, nb, stream=stream)
        else:
            P.relax_step(prm, src, dst, pr, li.owned, nb, stream=stream)
        evs[i][1].record(stream)
    stream.synchronize()
    k_ms = statistics.mean(a.elapsed_time(b) for a, b in evs[2:])
    halo = None
    if world > 1:
        halo = halo_metrics(halo_mode, n, ghost, tk, S, t_ms / args.steps, max_over_ranks(k_ms))
    variant = P.relax_variant(qa, qb, pr, li.owned)
    local_cells = (li.owned.hi.c[0] - li.owned.lo.c[0] + 1) * (li.owned.hi.c[1] - li.owned.lo.c[1] + 1)
    achieved = BYTES_PER_CELL_UPDATE * local_cells / (k_ms * 1e-3) / 1e9
    peak, peak_src = load_peaks()
    traffic = load_traffic(args.config) if world == 1 else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": (f"k_tbw<5pt,K={tk}> (temporal blocking, skewed wavefront: one launch = {tk} sweeps, "
                           f"{BYTES_PER_CELL_UPDATE}/{tk} B per cell-update)") if tk > 1 else
                          ("%s<RELAX,%s>%s" % ("k_bulk" if variant == 1 else "k_stream", "5pt" if cfg["stencil"] == 0
                                               else "9pt", " (TMA bulk-copy pipeline)" if variant == 1 else
                                               " (register-streaming LDG.128)")),
                "kernel_ms": k_ms, "algorithmic_bytes_per_launch": BYTES_PER_CELL_UPDATE * local_cells,
                "peak_source": peak_src, "whole_step_GBps": BYTES_PER_CELL_UPDATE * value}
    ceil = k12_ceiling(P, torch, dev, min(local_cells, 1 << 28), stream) if local_cells >= (1 << 22) else None
    roofline_extras(roofline, local_cells, ceil)
    if cfg.get("solve_kernel") and world == 1 and tk == 1:
        # small configs: px_solve runs the whole solve in one kernel whose iterate never
        # leaves the chip, so the timed step is that kernel; the fields above describe
        # a single k = 1 sweep launch for comparison with the large configs
        per_step = launches / args.steps
        kname = next((k for k in SOLVE_KERNELS if k in solve_kernels.split()), solve_kernels)
        roofline["solve_kernel"] = {
            "name": f"{kname} ({SOLVE_KERNELS.get(kname, 'whole solve in one launch')})",
            "launches_per_step": per_step, "ms_per_step": t_ms / args.steps,
            "us_per_sweep": 1e3 * t_ms / args.steps / S,
            "bound": "latency (on-chip iterate: block barriers and neighbour handshakes per sweep)",
            "equivalent_GBps_at_24B": BYTES_PER_CELL_UPDATE * value}

    # ---- end to end through the public host API (pinned host buffers; every
    # step's H2D of ρ and D2H of φ^N and its norms are inside the timed region).
    # N = 1: px_solve_host_batch, one problem per step, φ0 = 0 (NULL: zero-filled
    # on the device), copies of neighbouring steps overlapped with the solve.
    e2e = None
    if not args.no_e2e:
        ny = li.owned.hi.c[1] - li.owned.lo.c[1] + 1
        h_rho = lay.view(rank, rho if cfg["stencil"] == 0 else rhs).cpu().pin_memory()
        h_outs = [torch.empty((ny, n), dtype=torch.float64).pin_memory() for _ in range(2)]
        # a stream of problems: the first H2D and the last D2H of the pipeline
        # are not overlapped, so the e2e stream is 3x the timed steps (<= 30)
        ke = max(3, min(3 * args.steps, 30))
        if world == 1:
            e2e_norms = []

            def e2e_run(k):
                e2e_norms[:] = P.solve_host_batch(lay, prm, S, E, [h_rho.numpy()] * k,
                                                  [h_outs[i % 2].numpy() for i in range(k)], None,
                                                  use_graph=True, stream=stream, temporal_k=tk)
        else:
            # the bench's own (registered) buffers: φ0 and ρ copied in every step
            h_phi0 = torch.zeros((ny, n), dtype=torch.float64).pin_memory()
            h_out = h_outs[0]
            d_rhs = rho if cfg["stencil"] == 0 else rhs

            def e2e_step():
                with torch.cuda.stream(stream):
                    lay.view(rank, tens[0]).copy_(h_phi0, non_blocking=True)
                    lay.view(rank, d_rhs).copy_(h_rho, non_blocking=True)
                if tk > 1:
                    P.exchange_ghosts(lay, comm, rank, pr, stream=stream)
                r = P.solve(lay, scomm, rank, prm, S, E, bufs[0], bufs[1], pr, use_graph=True, stream=stream,
                            temporal_k=tk)
                with torch.cuda.stream(stream):
                    h_out.copy_(lay.view(rank, tens[1] if r.in_scratch else tens[0]), non_blocking=True)
                stream.synchronize()
                if r.in_scratch:
                    bufs.reverse()
                    tens.reverse()

            def e2e_run(k):
                for _ in range(k):
                    e2e_step()
        e2e_run(3)  # builds the plans / buffers of the three pipeline sets
        barrier()
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        e2e_run(ke)
        w1.record(stream)
        barrier()
        te_ms = max_over_ranks(w0.elapsed_time(w1))
        n_norm = (S + E - 1) // E + 1 if E > 0 else 1
        e2e = {"value": n * n * S * ke / (te_ms * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": (1 if world == 1 else 2) * n * n * 8,
               "d2h_bytes_per_step": n * n * 8 + 16 * n_norm, "steps": ke,
               "api": ("px_solve_host_batch (one problem per step: H2D rho, solve, D2H phi^N + norms; "
                       "phi0 = 0 zero-filled on the device; copies overlap the neighbouring steps' solves)")
               if world == 1 else f"torch pinned copies of phi0 and rho + px_solve ({halo_mode} halo) + D2H phi^N"}

    halo_proxy = None
    if world == 1 and tk == 1 and n >= 16384 and not args.no_halo_proxy and cfg["bc"] == 0:
        halo_proxy = measure_halo_proxy(P, torch, dev, stream, prm, n, 8, S)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # C1/C2 in full, C3/C5 at full size for >= 10 sweeps, C4 at 8192² (host RAM)
        n_s, sw = (n, 10) if n <= 16384 and n > 1024 else ((8192, 4) if n > 16384 else (n, S))
        r, dt = oracle_sample(cfg, n_s, sw)
        cpu = {"value": r, "unit": UNIT, "cores": 1, "kind": "oracle", "host": host_info(),
               "sample": f"single-threaded C++ oracle, {n_s}x{n_s} of the same recipe, {sw} sweeps, {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "n": n, "sweeps_per_step": S, "norm_every": E,
                       "temporal_k": tk, "ghost": ghost, "halo": halo_mode,
                       "steps_continue": "each step continues from the previous step's iterate",
                       "box": box, "partition": f"slabs x{world}", "rho": cfg["rho"], "h": h, "lambda": lam,
                       "l2": "inputs (3 x %.2f GB) exceed L2; no flush" % (lay.local(0).alloc_elems * 8 / 1e9)
                       if n >= 4096 else "L2-resident working set (no flush: that is the config)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk,
            "final_residual_max": float(d_norms.view(-1, 2)[res - 1, 0].item()) if res > 0 else None,
        }
        if halo is not None:
            line["halo"] = halo
        if halo_proxy is not None:
            line["halo_proxy"] = halo_proxy
        print(json.dumps(line))
    if scomm is not None and scomm is not comm:
        scomm.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def host_info() -> dict:
    """The GPU box's host: core count and CPU model (the oracle's context)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu": model}


def p2p_setup(P, torch, dist, lay, rank, world, local, comm, prm, S, pa, pb, pr, phi, stream):
    """The fused peer-memory push on a peer-memory communicator (records
    all-gathered over the torch process group), self-checked before use: a
    short solve from φ = 0 through the NCCL path and through the push path
    must give the same bits on every rank.  Returns (communicator, None) or
    (None, reason); φ is left zeroed."""
    def run(c):
        phi.zero_()
        torch.cuda.synchronize()
        r = P.solve(lay, c, rank, prm, 4, 1, pa, pb, pr, use_graph=False, stream=stream)
        return phi.clone(), r.norms.copy()
    try:
        ref, rn = run(comm)
        pcomm = P.Comm(None, world, rank, local)
        recs = [None] * world
        dist.all_gather_object(recs, P.comm_p2p_export(pcomm, lay, rank, pa, pb))
        P.comm_p2p_import(pcomm, lay, recs)
        got, gn = run(pcomm)
        ok = bool(torch.equal(lay.view(rank, got), lay.view(rank, ref))) and bool((gn[:, 0] == rn[:, 0]).all())
        why = "self-check differs from NCCL"
    except Exception as e:  # noqa: BLE001 -- reported in config.halo, the NCCL path runs instead
        pcomm, ok, why = None, False, f"{type(e).__name__}: {e}"[:200]
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=phi.device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    phi.zero_()
    torch.cuda.synchronize()
    if flag.item() == 1:
        return pcomm, None
    if pcomm is not None:
        pcomm.close()
    return None, why if not ok else "another rank's self-check failed"


def halo_metrics(mode, n, g, tk, S, ms_per_step, kernel_ms):
    """SURVEY §8(d) multi-GPU halo figures from the device-timed step and the
    sweep kernel alone (max over ranks).  Per sweep each rank sends g full
    padded rows to each of its two slab neighbours."""
    row_bytes = (n + 2 * g) * 8
    per_dir = g * row_bytes
    sweep_ms = ms_per_step / S * tk  # per exchange
    over_ms = max(sweep_ms - kernel_ms, 0.0)
    return {"path": mode, "bytes_per_neighbour_direction": per_dir, "bytes_sent_per_exchange_per_rank": 2 * per_dir,
            "exchange_every_sweeps": tk, "kernel_ms": kernel_ms, "ms_per_exchange_period": sweep_ms,
            "unoverlapped_us_per_exchange": 1e3 * over_ms, "unoverlapped_frac": over_ms / sweep_ms,
            "halo_GBps_per_direction_avg": per_dir / (sweep_ms * 1e-3) / 1e9,
            "nvlink_frac_of_900GBps": per_dir / (sweep_ms * 1e-3) / 900e9,
            "note": "push path: the halo stores are issued inside the sweep kernel, so the exchange has no span "
                    "of its own; the unoverlapped time is what the step adds over the sweep kernel alone"}


def measure_halo_proxy(P, torch, dev, stream, prm, n, p, S):
    """One-GPU proxy of the multi-GPU halo paths (N = 1 runs only): the slab
    of a p-rank split of the n² domain (n x n/p rows, periodic) solved for S
    sweeps with norms every sweep, graph replay, as (a) one rank with fused
    wrap images, (b) its own neighbour over NCCL send/recv (comm stream,
    boundary rows first) and (c) its own neighbour through the fused
    peer-memory push -- ms per sweep and overhead over the sweep kernel."""
    from paper_2307_07931_b200 import inputs
    os.environ["PROTOX_NCCL_SELF_EXCHANGE"] = "1"
    n1 = n // p
    lay = P.Layout(P.box(0, 0, n - 1, n1 - 1), (256, 256), 1, P.PX_BC_PERIODIC, 1)
    li = lay.local(0)
    a, b, r = lay.alloc(0, dev), lay.alloc(0, dev), lay.alloc(0, dev)
    stream.wait_stream(torch.cuda.current_stream(dev))
    P.init_field(lay, 0, lay.patch(0, r), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=stream)
    pa, pb, pr = lay.patch(0, a), lay.patch(0, b), lay.patch(0, r)
    nb = P.norm_buffer(li.owned, dev)
    stream.wait_stream(torch.cuda.current_stream(dev))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(23)]
    for i, (e0, e1) in enumerate(evs):
        src, dst = (pa, pb) if i % 2 == 0 else (pb, pa)
        e0.record(stream)
        P.relax_step(prm, src, dst, pr, li.owned, nb, stream=stream)
        e1.record(stream)
    stream.synchronize()
    out = {"slab": [n, n1], "ranks_emulated": p, "sweeps": S,
           "kernel_ms": statistics.mean(e0.elapsed_time(e1) for e0, e1 in evs[3:])}
    for mode in ("local", "nccl", "p2p"):
        comm = None
        if mode == "nccl":
            comm = P.Comm(P.comm_unique_id(), 1, 0, dev.index)
        elif mode == "p2p":
            comm = P.Comm(None, 1, 0, dev.index)
            P.comm_p2p_import(comm, lay, [P.comm_p2p_export(comm, lay, 0, pa, pb)])
        P.solve(lay, comm, 0, prm, S, 1, pa, pb, pr, use_graph=True, stream=stream)
        kern = P.last_solve_kernels()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            P.solve(lay, comm, 0, prm, S, 1, pa, pb, pr, use_graph=True, stream=stream)
        e1.record(stream)
        stream.synchronize()
        ms = e0.elapsed_time(e1) / (3 * S)
        out[mode] = {"ms_per_sweep": ms, "overhead_frac": ms / out["kernel_ms"] - 1, "sweep_kernels": kern}
        if comm is not None:
            comm.close()
    P.release_cached()
    del a, b, r
    torch.cuda.empty_cache()
    return out


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def ensure_ranks(args):
    """One process per GPU.  Under torchrun WORLD_SIZE must equal --gpus.
    Outside torchrun, --gpus N > 1 re-launches this script under
    torch.distributed.run with N ranks (127.0.0.1) and returns its exit code,
    so a scaling run can never silently measure one rank; the native arm
    refuses (exit 2) when fewer than N GPUs are visible.  Returns None when the
    current process should run the benchmark itself."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
            return 2
        return None
    if args.gpus <= 1:
        return None
    if args.impl == "native":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}; "
                             "refusing to measure fewer ranks\n")
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    sys.stderr.write("bench.py: launching %d ranks: %s\n" % (args.gpus, " ".join(cmd)))
    sys.stderr.flush()
    return subprocess.call(cmd)


def main():
    args = parse()
    rc = ensure_ranks(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    if CONFIGS[args.config].get("dims") == 3:
        return run_native3d(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
