"""Multi-GPU tier: one process per GPU over CUDA-IPC/NVLink, each rank checked
against the golden fixtures and the oracle (tests/mp_worker.py)."""

import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(n):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mp_worker.py")]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    proc = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    out = proc.stdout + proc.stderr
    assert proc.returncode == 0, out[-6000:]
    assert out.count("checks passed") == n, out[-3000:]


@pytest.mark.gpu
@pytest.mark.multigpu(2)
def test_two_gpus():
    _run(2)


@pytest.mark.gpu
@pytest.mark.multigpu(4)
def test_four_gpus():
    _run(4)


@pytest.mark.gpu
@pytest.mark.multigpu(8)
def test_eight_gpus():
    _run(min(8, torch.cuda.device_count()))
