"""bench.py's reference arm (the oracle on the host cores, tier rules ④) keeps the
driver's JSON-line contract: one line from rank 0, the metric and unit of
BASELINE.json, a cpu_baseline of kind "oracle", an e2e object with zero copy bytes.
Under torchrun with two ranks only rank 0 prints; the other exits 0 without work."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def _check(line, config_desc_key="workload"):
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert line["impl"] == "reference"
    assert line["metric"] == base["metric"]
    assert line["unit"] == "Gcell-updates/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["warmup"] >= 3 and line["steps"] >= 1
    assert line["dtype"] == "f64" and line["data"] == "synthetic"
    assert config_desc_key in line["config"] and "sample" in line["config"]
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    e = line["e2e"]
    assert e["value"] == line["value"] and e["unit"] == line["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


@pytest.mark.parametrize("config", ["C1", "C3D"])
def test_reference_arm_line(config):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", config,
                        "--steps", "1", "--warmup", "3"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _lines(p.stdout)
    assert len(lines) == 1
    _check(lines[0])
    assert lines[0]["n_gpus"] == 1


def test_reference_arm_torchrun_two_ranks():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29631", "bench.py", "--impl",
                        "reference", "--config", "C1", "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _lines(p.stdout)
    assert len(lines) == 1  # rank 0 only
    _check(lines[0])
    assert lines[0]["n_gpus"] == 2


def test_native_arm_fails_loudly_without_gpu():
    """The product path has no CPU fallback: with no GPU the native arm exits non-zero
    and prints no bench line."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, "bench.py", "--steps", "1", "--warmup", "3"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode != 0
    assert _lines(p.stdout) == []


def test_binding_raises_when_library_missing(monkeypatch):
    from paper_2307_07931_b200 import protox as P
    monkeypatch.setattr(P, "_lib", None)
    monkeypatch.setattr(P, "LIB_PATH", os.path.join(ROOT, "no_such_dir", "libprotox.so"))
    with pytest.raises(RuntimeError, match="not built"):
        P.lib()


def test_gpus_flag_spawns_ranks_itself():
    """`bench.py --gpus 2` outside torchrun re-launches itself with two ranks
    (torch.distributed.run): the reference arm (no GPU needed) then prints one
    line from rank 0 with n_gpus = 2 -- never a silent one-rank measurement."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C1", "--gpus", "2",
                        "--steps", "1", "--warmup", "3"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "launching 2 ranks" in p.stderr
    lines = _lines(p.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2


def test_native_multi_gpu_refuses_without_enough_gpus():
    """The native arm with --gpus 2 and fewer visible GPUs exits non-zero with
    a message and no bench line."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "3"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 2
    assert "refusing" in p.stderr
    assert _lines(p.stdout) == []


def test_world_size_mismatch_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0", CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--impl", "reference", "--config", "C1"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 2 and "WORLD_SIZE" in p.stderr
