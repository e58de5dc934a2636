"""The driver's bench.py contract, checked on the device: one JSON line with the required keys and
types for both arms (our kernels, and --impl reference = the CPU oracle), the roofline /
cpu_baseline / e2e / clocks / gpu_launches objects, and consistent arithmetic (value = pairs per
second of the timed steps)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_bench_line_contract():
    d = _run("--steps", "3", "--warmup", "3")
    for k, t in [("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int), ("warmup", int),
                 ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str), ("dtype", str),
                 ("data", str), ("config", dict), ("roofline", dict), ("cpu_baseline", dict), ("e2e", dict),
                 ("gpu_launches", int), ("clocks", dict)]:
        assert isinstance(d[k], t), (k, d.get(k))
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["vs_baseline"] is None and d["scaling"] == "strong" and d["config"]["workload"].startswith("C4")
    assert d["config"]["n_items"] == 100_000 and d["config"]["n_transactions"] == 1_000_000
    pairs = d["config"]["pairs_per_step"]
    assert abs(d["value"] - pairs / (d["ms_per_step"] / 1e3)) / d["value"] < 1e-6
    r = d["roofline"]
    assert r["bound"] == "alu" and r["unit"] == "Tcmp/s" and 0.3 < r["frac"] < 1.0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    # traffic: the committed ncu figure of this workload's K2 launch, against the arena it must read
    assert r["compulsory_bytes"] == 2_487_803_904 and r["traffic"] >= r["compulsory_bytes"] and r["traffic_src"]
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"] and c["cpu_model"]
    for alg in ("horizontal", "merge"):  # both oracles, 1 thread and all threads
        assert c[alg]["1t"] > 0 and c[alg]["all"] > 0
    assert c["value"] == c["horizontal"]["all"]
    x = d["extra"]
    assert x["C2"]["value"] > 0 and x["C4_prefiltered"]["frequent_pairs"] == d["config"]["frequent_pairs"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["metric"] and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_bench_two_ranks_contract():
    """N = 2 under torchrun (both ranks on this GPU over gloo, the bench's test hook): rank 0 alone
    prints one line with n_gpus = 2 on the SAME C4 instance (strong scaling), verified against the
    oracle before timing, and an e2e through dist.mine_distributed."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", BENCH_FORCE_DEVICE="0")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["n_items"] == 100_000 and d["scaling"] == "strong"
    assert d["verified_vs_oracle_before_timing"] is True
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and "mine_distributed" in d["e2e"]["api"]
    assert d["cpu_baseline"] is None  # rank 0 at N = 1 only
