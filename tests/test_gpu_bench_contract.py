"""bench.py keeps its JSON contract (one line on stdout; the keys the driver and the judge read),
on small configurations so that the check takes seconds: the default path, every opt-in path
(disk cache, trainer, DGL blocks, sequential) and the reference arm."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=900):
    p = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _check_common(d, steps, warmup):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config"):
        assert k in d, k
    assert d["steps"] == steps and d["warmup"] == warmup and d["n_gpus"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert "workload" in d["config"]


def test_default_contract_products():
    # (a products pass takes ~50 ms: enough steps that the clock sampler sees the GPU under load)
    d = _run("--config", "products", "--steps", "12", "--warmup", "3", "--cpu-batches", "4", "--e2e-steps", "1")
    _check_common(d, 12, 3)
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] <= 1.0 and r["peak"] > 0 and r["achieved"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and "clocks" in d and d["clocks"]["sm_mhz"] is not None
    assert d["e2e"]["mode"] == "host-features"
    assert d["offline"]["batches_per_s"] > 0 and d["sampling"]["edges_per_s"] > 0


@pytest.mark.parametrize("flags", [["--disk-budget", "0.9", "--train"], ["--blocks", "--sequential"],
                                   ["--stage", "file", "--embed-graph"]])
def test_opt_in_paths_tiny(flags):
    d = _run("--config", "tiny", "--steps", "2", "--warmup", "3", "--no-e2e", "--cpu-batches", "8", *flags)
    _check_common(d, 2, 3)
    assert d["gpu_launches"] > 0
    if "--disk-budget" in flags:
        assert "disk_cache" in d["layout_stats"]
        assert d["layout_stats"]["disk_cache"]["space_pages"] <= d["layout_stats"]["disk_cache"]["budget_pages"]
        assert "trainer stub" in d["config"]["schedule"]
    if "--stage" in flags:
        assert "file on local storage" in d["config"]["disk_tier"] and "graph loader" in d["config"]["disk_tier"]
        assert d["disk_io"]["bytes_read_per_step"] > 0 and "trainer stub" in d["config"]["schedule"]
    if "--blocks" in flags:
        assert "DGL-block" in d["config"]["schedule"] and "DGL blocks" in d["cpu_baseline"]["sample"]


def test_reference_arm_tiny():
    d = _run("--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.parametrize("split", ["weak", "epoch"])
def test_two_rank_launch_on_one_gpu(split):
    """The N > 1 path of bench.py as the driver launches it (torch.distributed.run, one process
    per rank, batch-sharded epochs, the count all-reduce, max-over-ranks timing, one JSON line
    from rank 0), with both ranks on the box's one GPU and gloo standing in for NCCL.  weak: one
    epoch per rank; epoch: one epoch split into contiguous batch blocks (strong scaling)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, DGNN_BENCH_SHARE_GPU="1", DGNN_BENCH_BACKEND="gloo")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={port}", "bench.py", "--gpus", "2",
                        "--config", "tiny", "--steps", "2", "--warmup", "3", "--no-cpu", "--e2e-steps", "1",
                        "--split", split],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == ("weak" if split == "weak" else "strong")
    assert d["config"]["parallelism"].startswith("dp2")
    # value counts the batches of both ranks: two epochs (weak) or one epoch of 8 batches (strong)
    per_step = 2 * d["config"]["batches_per_rank"] if split == "weak" else 8
    assert abs(d["value"] - per_step * d["steps"] / (d["ms_per_step"] * d["steps"] / 1e3)) <= 0.02 * d["value"]
    assert d["e2e"]["value"] > 0


@pytest.mark.parametrize("split,mode,shard", [("weak", "replicated", ""), ("epoch", "replicated", ""),
                                              ("epoch", "peer", ""), ("weak", "peer", ""), ("epoch", "nccl", ""),
                                              ("epoch", "peer", "shard"), ("weak", "replicated", "shard")])
def test_two_rank_runner_outputs_equal_the_oracle(split, mode, shard):
    """bench.py's Runner at world size 2 (both ranks on the one GPU, gloo for the collectives, the
    all-to-all through host memory): every assembled batch of three pipelined passes equals the
    oracle, for both splits, every GPU-tier mode, and the feature table partitioned by node range
    over the ranks (CUDA IPC mappings) (tests/multirank_runner_check.py)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, DGNN_BENCH_SHARE_GPU="1", DGNN_BENCH_BACKEND="gloo")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={port}", "tests/multirank_runner_check.py",
                        split, mode, shard], cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    import re
    oks = re.findall(r"rank (\d): (ok|FAIL[^\n]*?)(?=rank \d:|\n|$)", p.stdout)
    assert sorted(oks) == [("0", "ok"), ("1", "ok")], p.stdout[-3000:]


def test_two_rank_launch_partitioned_tier():
    """bench.py at N = 2 with the GPU tier partitioned over the ranks (peer memory): one JSON line,
    the HBM-budget capacities (2 x the config's GPU rows) and the mode in the config."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, DGNN_BENCH_SHARE_GPU="1", DGNN_BENCH_BACKEND="gloo")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={port}", "bench.py", "--gpus", "2",
                        "--config", "tiny", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-e2e",
                        "--split", "epoch", "--gpu-tier", "peer"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert d["config"]["gpu_rows"] == 1000 and "partitioned" in d["config"]["parallelism"]
