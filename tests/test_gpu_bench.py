"""bench.py end to end on the GPU box, at small sizes: the JSON line keeps the driver's
contract (keys, units, launches, roofline, cpu_baseline, e2e, clocks) at N = 1; the shot
sharding runs under torchrun with the test-only overrides BENCH_ONE_DEVICE (every rank on
device 0) and BENCH_DIST_BACKEND=gloo (no collective on the data path: the ranks never wait
on one another's kernels); the band decomposition runs as --dist-local ranks on one GPU.
Functional checks, never a reported number."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run(args, nproc=1, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    if nproc > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), "bench.py"] + args
    else:
        cmd = [sys.executable, "bench.py"] + args
    o = subprocess.run(cmd, cwd=ROOT, env=e, capture_output=True, text=True, timeout=timeout)
    assert o.returncode == 0, o.stderr[-2000:]
    lines = [l for l in o.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, o.stdout[-2000:]
    return json.loads(lines[0])


def check_line(d, n_gpus, scaling):
    assert d["metric"].startswith("fp64 grid-point updates/sec")
    assert d["unit"] == "grid-point updates/s" and d["value"] > 0 and d["ms_per_step"] > 0
    assert d["n_gpus"] == n_gpus and d["scaling"] == scaling and d["dtype"] == "f64"
    assert d["higher_is_better"] is True and d["data"] == "synthetic"
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["roofline_fp64"]["achieved"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_bench_one_gpu_contract():
    d = run(["--grid", "2049", "--steps", "3", "--warmup", "3", "--cpu-n", "257"])
    check_line(d, 1, "strong")
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert set(d["per_method"]) == {"mfd", "cfd"}


def test_bench_reference_arm():
    d = run(["--impl", "reference", "--steps", "1", "--warmup", "3", "--cpu-n", "257"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def test_bench_band_decomposition_one_gpu():
    """bench.py --gpus N runs adi_create_dist (NCCL between GPUs; one GPU per rank, so not
    runnable here); --dist-local P runs the same library path with the loopback transport,
    P ranks on this GPU."""
    for mode in ("halo", "transpose"):
        d = run(["--dist-local", "3", "--dist-mode", mode, "--grid", "2049", "--steps", "2", "--warmup", "3",
                 "--no-cpu"])
        check_line(d, 1, "strong")
        assert "adi_create_dist_local" in d["config"]["parallelism"] and mode in d["config"]["parallelism"]


def test_bench_shots_two_ranks():
    env = {"BENCH_ONE_DEVICE": "1", "BENCH_DIST_BACKEND": "gloo"}
    d = run(["--shots", "--shots-per-gpu", "2", "--gpus", "2", "--steps", "3", "--warmup", "3"], nproc=2, env=env)
    check_line(d, 2, "weak")
    assert d["config"]["shots_total"] == 4 and d["e2e"]["value"] > 0
