"""Measured algorithm-selection table (BASELINE north_star: "the choice is
made by a size threshold measured on the box").

``tuning.json`` next to this file is written by ``bench.py --tune`` on a B200
box: for every group size it stores the message size from which ring_rsa
(two-shot reduce-scatter + allgather) beats rhd_rsa (one-shot tree), the
largest message worth reducing one-shot and the largest worth the LL
two-shot. Without an entry the reference default of 131072 B
(collectives.py:23) applies.
"""

from __future__ import annotations

import json
import os
from functools import lru_cache

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tuning.json")
DEFAULT_SWITCH_BYTES = 131072


@lru_cache(maxsize=1)
def table() -> dict:
    try:
        with open(PATH) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def switch_bytes_for(p: int) -> int:
    return int(table().get("switch_bytes", {}).get(str(p), DEFAULT_SWITCH_BYTES))


def oneshot_max_for(p: int) -> int | None:
    v = table().get("oneshot_max_bytes", {}).get(str(p))
    return None if v is None else int(v)


def ll2_max_for(p: int) -> int | None:
    """Largest message worth the LL two-shot kernel (above it: the pull
    two-shot); None = the kernel's own limit (p x the LL slot payload)."""
    v = table().get("ll2_max_bytes", {}).get(str(p))
    return None if v is None else int(v)
