"""Restatement of the pointer-cache registry semantics — TEST INFRASTRUCTURE.

Restates ``/root/reference/pkg/src/collectium/registry.py:52-151`` as a trace
replayer: given an op trace it returns every classify answer and the final
``RegistryStats`` per policy.  The product's C++ registry
(``paper_1810_11112_b200/csrc/ptrcache.cpp``) is checked against this and
against golden traces generated from the reference.
"""

from __future__ import annotations

import heapq

BASE_ADDRESS = 0x1000                                         # registry.py:20


def replay(trace, policy: str):
    """trace items: ("alloc", idx, kind, size) | ("free", idx) |
    ("classify", idx) | ("classify_addr", address).  Returns (answers,
    stats dict, addresses by idx).  Errors are recorded as the answer
    strings "InvalidHandleError"/"UnknownBufferError"."""
    live, kinds, cache = {}, {}, {}
    freed: list[int] = []
    nxt = BASE_ADDRESS
    st = dict(driver_queries=0, cache_hits=0, inserts=0, invalidations=0)
    addr_of = {}
    answers = []

    def driver(a):
        st["driver_queries"] += 1
        if a not in kinds:
            return "UnknownBufferError"
        return kinds[a]

    for op in trace:
        if op[0] == "alloc":
            _, idx, kind, size = op
            if freed:
                a = heapq.heappop(freed)                      # registry.py:75-79
            else:
                a, nxt = nxt, nxt + 1
            live[a] = idx
            kinds[a] = kind
            addr_of[idx] = a
            if policy == "intercept_cache":
                cache[a] = kind
                st["inserts"] += 1
        elif op[0] == "free":
            a = addr_of.get(op[1])
            if a is None or live.get(a) != op[1]:
                answers.append("InvalidHandleError")
                continue
            del live[a]
            del kinds[a]
            heapq.heappush(freed, a)
            if policy == "intercept_cache":
                del cache[a]
                st["invalidations"] += 1
        else:
            a = addr_of[op[1]] if op[0] == "classify" else op[1]
            if policy == "no_cache":
                answers.append(driver(a))
            elif policy == "lazy_cache":
                if a in cache:
                    st["cache_hits"] += 1
                    answers.append(cache[a])
                else:
                    k = driver(a)
                    if k != "UnknownBufferError":
                        cache[a] = k
                        st["inserts"] += 1
                    answers.append(k)
            else:
                if a not in cache:
                    answers.append("UnknownBufferError")
                else:
                    st["cache_hits"] += 1
                    answers.append(cache[a])
    return answers, st, addr_of
