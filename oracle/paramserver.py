"""Numpy restatement of the parameter-server pull step — TEST INFRASTRUCTURE.

Restates ``/root/reference/pkg/src/collectium/paramserver.py``:
``PsTopology.create`` (:159-165, round-robin shard map over the PS ranks in
sorted name order) and the arithmetic of ``run_ps_step`` (:171-271): each
owner sums the workers' gradient shards in worker-rank order in float64,
divides by the worker count, and applies ``param - lr * mean`` in float64
before casting back to the parameter dtype; every worker ends with the
owners' updated shards.
"""

from __future__ import annotations

import numpy as np


def shard_map(names, ps_ranks) -> dict:
    """paramserver.py:159-165."""
    ps = sorted(ps_ranks)
    return {name: ps[i % len(ps)] for i, name in enumerate(sorted(names))}


def ps_step(grads_per_worker: list, params: dict, workers, lr: float) -> dict:
    """paramserver.py:214-229 (the owner's update; identical on every worker
    after the pull). ``grads_per_worker[i]`` is worker ``sorted(workers)[i]``'s
    {name: array}; returns {name: updated array}."""
    out = {}
    for name in sorted(params):
        contrib = [g[name] for g in grads_per_worker]
        acc = contrib[0].astype(np.float64)
        for c in contrib[1:]:
            acc = acc + c
        mean = acc / len(contrib)
        p = params[name]
        out[name] = (p.astype(np.float64) - lr * mean).astype(p.dtype)
    return out
