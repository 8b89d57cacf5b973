"""Load the committed golden fixtures (tests/golden/golden.json)."""
import json
import os
from functools import lru_cache

HERE = os.path.dirname(os.path.abspath(__file__))


@lru_cache(maxsize=1)
def cases():
    with open(os.path.join(HERE, "golden.json")) as fh:
        return json.load(fh)["cases"]


def of_kind(kind):
    return [c for c in cases() if c["kind"] == kind]
