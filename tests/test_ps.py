"""Parameter-server pull step (paramserver.py:159-271).

CPU: the numpy restatement (oracle/paramserver.py) reproduces the unmodified
reference's results (tests/golden/ps.json, from tests/golden/gen_sweep.py
--ps). GPU: the NVLink step (cm_ps_step, one kernel per rank) on a
single-GPU VirtualGroup is bit-identical to both."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import paramserver as OPS

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ps.json")))


def case_inputs(c):
    """Same draws as gen_sweep.py ps_cases(): params, then each worker's grads."""
    rng = np.random.default_rng(c["seed"])
    names = [f"w{i:02d}" for i in range(len(c["sizes"]))]
    params = {nm: rng.standard_normal(n).astype(c["dtype"]) for nm, n in zip(names, c["sizes"])}
    grads = [{nm: rng.standard_normal(n).astype(c["dtype"]) for nm, n in zip(names, c["sizes"])}
             for _ in c["workers"]]
    return names, params, grads


@pytest.mark.parametrize("c", CASES, ids=lambda c: f"w{c['workers']}-ps{c['ps']}-{c['dtype']}")
def test_oracle_matches_reference_golden(c):
    names, params, grads = case_inputs(c)
    out = OPS.ps_step(grads, params, c["workers"], c["lr"])
    assert {k: hashlib.sha256(v.tobytes()).hexdigest() for k, v in out.items()} == c["sha"]
    smap = OPS.shard_map(names, c["ps"])
    assert sorted(set(smap.values())) == sorted(set(c["ps"]) & set(smap.values()))


@pytest.mark.gpu
@pytest.mark.parametrize("c", CASES, ids=lambda c: f"w{c['workers']}-ps{c['ps']}-{c['dtype']}")
def test_nvlink_ps_step_virtual_bit_exact(c):
    import torch
    import paper_1810_11112_b200 as P
    names, params, grads = case_inputs(c)
    p = max(max(c["workers"]), max(c["ps"])) + 1
    vg = P.VirtualGroup(p, 0, staging_bytes=16 << 20, timeout_s=5.0)
    topo = P.PsTopology.create(c["workers"], c["ps"], names)
    ptensors = [P.Tensor(nm, c["dtype"], torch.from_numpy(params[nm]).cuda()) for nm in names]
    gper = [None] * p
    for i, w in enumerate(c["workers"]):
        gper[w] = [P.Tensor(nm, c["dtype"], torch.from_numpy(grads[i][nm]).cuda()) for nm in names]
    for _ in range(2):          # both staging parities
        res = P.run_ps_step_group(vg, topo, gper, [ptensors] * p, c["lr"])
        for r in range(p):
            if r in c["workers"]:
                assert {t.name: hashlib.sha256(t.to_bytes()).hexdigest() for t in res[r]} == c["sha"], r
            else:
                assert res[r] is None
    vg.close()


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 5, 8])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_nvlink_ps_step_virtual_large_vs_oracle(p, dtype):
    """Large tensors reach the owner phase's unrolled loop (>= 4 x 512
    elements per CTA piece, for float64 too) and, with a schema whose total is
    not a multiple of 4 elements, a served area that starts 16-byte aligned."""
    import torch
    import paper_1810_11112_b200 as P
    rng = np.random.default_rng([p, 7])
    sizes = [300_001, 17, 1 << 20, 4096, 99_999, 2]
    names = [f"layer{i:03d}" for i in range(len(sizes))]
    params = {nm: rng.standard_normal(n).astype(dtype) for nm, n in zip(names, sizes)}
    grads = [{nm: rng.standard_normal(n).astype(dtype) for nm, n in zip(names, sizes)} for _ in range(p)]
    want = OPS.ps_step(grads, params, list(range(p)), 0.1)
    vg = P.VirtualGroup(p, 0, staging_bytes=32 << 20, timeout_s=5.0)
    topo = P.PsTopology.create(range(p), range(p), names)
    pt = [P.Tensor(nm, dtype, torch.from_numpy(params[nm]).cuda()) for nm in names]
    gper = [[P.Tensor(nm, dtype, torch.from_numpy(grads[r][nm]).cuda()) for nm in names] for r in range(p)]
    res = P.run_ps_step_group(vg, topo, gper, [pt] * p, 0.1)
    for r in range(p):
        assert all(t.to_bytes() == want[t.name].tobytes() for t in res[r])
    vg.close()
