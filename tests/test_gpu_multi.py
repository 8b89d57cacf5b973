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


def _run(n, extra_env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mp_worker.py")]
    env = dict(os.environ, OMP_NUM_THREADS="1", **(extra_env or {}))
    proc = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    out = proc.stdout + proc.stderr
    assert proc.returncode == 0, out[-6000:]
    assert out.count("checks passed") == n, out[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_ranks_sharing_one_gpu(n):
    """The real multi-process communicator (CUDA-IPC heaps, NVLink flag
    protocol, cm_fused_allreduce_agreed, cm_agree, registration, the host
    pipeline, the parameter server) with n processes on ONE GPU: IPC handles
    open within a device too, and the contexts' kernels interleave, so every
    cross-process path of the N-GPU tier runs on a single-GPU box."""
    _run(n, {"CUDA_VISIBLE_DEVICES": os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0]})


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


@pytest.mark.gpu
def test_cli_microbench_and_train_two_ranks(tmp_path):
    """The reference-format harness (cli.py) under torchrun: CSV header and
    rows as collectium writes them, plus the B200 columns."""
    out = tmp_path / "micro.csv"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           "-m", "paper_1810_11112_b200.cli", "--mode", "microbench", "--msg-min-bytes", "8",
           "--msg-max-bytes", "1048576", "--warmup-iters", "2", "--timed-iters", "5", "--output", str(out)]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    proc = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, (proc.stdout + proc.stderr)[-4000:]
    rows = out.read_text().splitlines()
    assert rows[0] == ("message_bytes,algo,p,mean_latency_s,min_latency_s,max_latency_s,messages_per_rank,"
                       "device_latency_s,bus_gbps,roofline_frac")
    assert len(rows) == 1 + 18                       # 8 B .. 1 MiB
    for r in rows[1:]:
        f = r.split(",")
        size, algo, p = int(f[0]), f[1], int(f[2])
        assert p == 2 and algo == ("rhd_rsa" if size < 131072 else "ring_rsa")
        assert int(f[6]) == 2                        # messages_per_rank, reference schedule at p=2
        assert 0 < float(f[4]) <= float(f[3]) <= float(f[5])
    out2 = tmp_path / "train.csv"
    dump = tmp_path / "final.npz"
    cmd = cmd[:cmd.index("--mode")] + ["--mode", "train", "--model", "mobilenet_like", "--warmup-iters", "1",
                                        "--timed-iters", "2", "--output", str(out2), "--dump-grads", str(dump)]
    cmd[cmd.index("--master-port") + 1] = str(_free_port())
    proc = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, (proc.stdout + proc.stderr)[-4000:]
    rows = out2.read_text().splitlines()
    assert rows[0] == "model,strategy,p,images_per_sec,ideal,efficiency"
    f = rows[1].split(",")
    assert f[:3] == ["mobilenet_like", "horovod_allreduce", "2"] and 0 < float(f[5]) <= 1.0
    # acceptance criterion 9 analogue (test_acceptance.py:331-366): the final
    # data-path tensors equal the reference's aggregate of the same synthetic
    # gradients (last iteration), bit for bit
    import numpy as np
    from oracle import aggregation as OA
    from tests.golden import inputs as I
    last = 1 + 2 - 1
    per_rank = [I.synth_gradients(0, last, I.MODELS["mobilenet_like"], r) for r in range(2)]
    want, _, _ = OA.aggregate(per_rank, "float32", "auto", 64 << 20)
    got = np.load(dump)
    assert sorted(got.files) == sorted(want)
    assert all(got[k].tobytes() == want[k].tobytes() for k in want)
    # ps_pull strategy: the parameter-server path, params from zeros, lr 0.1
    from oracle import paramserver as OPS
    cmd[cmd.index("--master-port") + 1] = str(_free_port())
    i = cmd.index("--output")
    cmd = cmd[:i] + ["--output", str(out2), "--dump-grads", str(dump), "--strategy", "ps_pull"]
    proc = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, (proc.stdout + proc.stderr)[-4000:]
    assert out2.read_text().splitlines()[1].split(",")[1] == "ps_pull"
    names = [nm for nm, _ in per_rank[0]]
    cur = {nm: np.zeros(a.size, np.float32) for nm, a in per_rank[0]}
    for it in range(3):
        grads = [dict(I.synth_gradients(0, it, I.MODELS["mobilenet_like"], r)) for r in range(2)]
        cur = OPS.ps_step(grads, cur, [0, 1], 0.1)
    got = np.load(dump)
    assert all(got[k].tobytes() == cur[k].tobytes() for k in names)
