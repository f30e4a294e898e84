"""bench.py's torchrun (N > 1) path end to end on ONE GPU: two ranks share
device 0 on a 1-GPU box (SDP_BENCH_SAME_DEVICE; ranks take GPUs round-robin when
several are visible), plumbing over gloo, data path over CUDA IPC
with the cross-rank flag barriers.  Timing is meaningless here (the two
processes' kernels are time-sliced); the test checks the path runs and emits
the contract's JSON line."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_torchrun_two_ranks_same_device(cuda):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, SDP_BENCH_SAME_DEVICE="1", SDP_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "5", "--warmup", "3", "--train-steps", "2", "--workload", "resnet18"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["gpu_launches"] == 5 and d["value"] > 0
    assert "nvlink_frac" in d["roofline"] and d["roofline"]["p2p_copy_GBps_measured"] > 0
    assert d["roofline"]["busbw_GBps"] > 0 and "busbw_frac_900" in d["roofline"] and "busbw_frac_probe" in d["roofline"]
    t = d["train"]  # PeerTrainer at world 2: C2 / C3 / DP samples/s and memory
    assert t["subnet_samples_per_s_per_gpu"] > 0 and t["widthwise_samples_per_s_per_gpu"] > 0
    assert t["subnet_peak_mem_per_gpu_bytes"] < t["dp_peak_mem_per_gpu_bytes"]
    assert t["c4_gpt2"]["subnet_tokens_per_s_per_gpu"] > 0 and t["c4_gpt2"]["dp_tokens_per_s_per_gpu"] > 0
