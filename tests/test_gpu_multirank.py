"""The N>1 bench path (paper Alg. 2: partition_by_ops ranges, per-rank GPU
range products, the rank-ordered gather by peer copies through CUDA IPC or by
an all-gather) run as 2 and 3 torchrun ranks that
share cuda:0 over gloo; the assembled product must carry the reference digest.
(The real N-GPU run uses NCCL; only one GPU is available to the tests.)"""

from __future__ import annotations

import json
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("ranks,config,gather", [(2, "fateman10", "peer"), (3, "fateman20", "peer"),
                                                 (2, "mp12", "peer"), (2, "fateman10", "collective"),
                                                 (3, "mp12", "collective"), (8, "mp12", "peer")])
def test_emulated_ranks_reproduce_reference_digest(ranks, config, gather):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", str(ROOT / "bench.py"),
           "--gpus", str(ranks), "--config", config, "--steps", "1", "--warmup", "1",
           "--emulate-ranks", "--verify", "--gather", gather]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    v = lines[0]["verified"]
    assert v["ok"], v


def test_bench_self_launches_ranks_without_torchrun():
    """`bench.py --gpus 3` with no torchrun: it launches the 3 ranks itself (one
    process per GPU; emulated over gloo when fewer devices are visible), and
    rank 0 prints one line with n_gpus 3, e2e and the verified product."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "3", "--config", "fateman20", "--steps", "1",
           "--warmup", "1", "--verify", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    v = lines[0]
    assert v["n_gpus"] == 3 and v["verified"]["ok"], v.get("verified")
    assert v["e2e"]["value"] > 0 and v["e2e"]["d2h_bytes_per_step"] > 0
    assert "gather_ms" in v["multi_gpu"] and "gather" in v["roofline"]["phases_ms"]


@pytest.mark.parametrize("ranks,cfg", [(2, "fateman10/int"), (3, "mp12/int"), (2, "fateman10/float")])
def test_gpu_mul_api_peer_gather(ranks, cfg):
    """cluster.gpu_mul (the multi-GPU public API) over emulated ranks: range
    products on the GPU, peer-copy gather, reference digest."""
    from conftest import digests
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", str(ROOT / "tests" / "multirank_api.py"), cfg]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    got = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")][0]
    want = digests()["products"][cfg]
    assert got["n"] == want["n"] and got["sha256"] == want["sha256"] and got["type"] == "Polynomial"
