"""Multi-process (one process per GPU part) path on a single GPU.

Two processes each own one part; their solve kernels synchronise only
through the CUDA-IPC peer-memory flag protocol (the contexts time-slice on
one GPU, which makes races far more likely than over NVLink).  The result
must be bit-identical to the single-process team, and the torchrun bench
path must run end to end.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_processes_bit_identical_to_single_process():
    env = dict(os.environ, LRB_BARRIER_TIMEOUT_S="30")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ipc_selftest.py")],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1]
    out = json.loads(line)
    assert res.returncode == 0, (res.stdout[-2000:], res.stderr[-2000:])
    assert out["bit_identical"] and out["ipc_iterations"] == out["single_iterations"]


def test_torchrun_bench_two_ranks_on_one_gpu():
    env = dict(os.environ, LRB_BARRIER_TIMEOUT_S="60")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29731", "bench.py", "--gpus", "2",
           "--workload", "c1", "--steps", "3", "--warmup", "3"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["gpu_launches"] > 0
    # both processes ran the team kernel; plumbing over gloo (they share the GPU)
    assert line["devices_ran_solve"] == 2 and len(line["per_device"]) == 2
    assert "gloo" in line["plumbing"]


def _torchrun(args, port):
    env = dict(os.environ, LRB_BARRIER_TIMEOUT_S="60")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", *args]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]   # rank 0 alone prints
    return lines[0]


def test_torchrun_c5_update_only_two_ranks():
    line = _torchrun(["--gpus", "2", "--workload", "c5", "--steps", "3", "--warmup", "3",
                      "--no-pageable"], 29733)
    assert line["n_gpus"] == 2 and line["config"]["parts_per_gpu"] == 4
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0


def test_torchrun_reference_arm_rank0_only():
    line = _torchrun(["--impl", "reference", "--gpus", "2", "--workload", "c1", "--steps", "1",
                      "--warmup", "3"], 29735)
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["cores"] >= 1
