"""CPU tier: the C-ABI library loads, exports every symbol include/cm.h
declares, and its host-side logic (chunking, layouts, algorithm selection,
reference CollectiveStats, fusion plan, simulated pointer cache) matches the
golden fixtures and the oracle. No kernel is launched here."""

import json
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_1810_11112_b200 as P
from paper_1810_11112_b200 import _lib as L
from oracle import aggregation as OA
from oracle import collectives as OC
from oracle import registry as OR
from tests.golden import inputs as I
from tests.golden.load import of_kind

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "cm.h")).read()
    declared = set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(cm_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 45
    for name in declared:
        assert hasattr(L.lib, name), name
    assert declared == set(L.EXPORTS), declared ^ set(L.EXPORTS)
    assert b"sm_100a" in L.lib.cm_version()


def test_fast_call_module_is_bound_to_the_loaded_library():
    """csrc/pyfast.cpp: built next to libcm.so and bound to the entry points
    of the same library instance; argument errors raise, not crash."""
    if os.environ.get("CM_NO_FAST"):
        pytest.skip("fast-call path disabled")
    assert L.fast is not None, "the _cmfast module is not built (python paper_1810_11112_b200/_build.py)"
    with pytest.raises(TypeError):
        L.fast.allreduce(1, 2, 3)
    with pytest.raises(TypeError):
        L.fast.fused(*range(14))
    with pytest.raises(TypeError):
        L.fast.sync(0)
    with pytest.raises(OverflowError):
        L.fast.allreduce(-1, 0, 0, 0, 0, 0, 0, 0, 0, 0)


def test_library_is_sm100a_build():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("p", range(1, 17))
def test_chunk_partition_and_layouts_match_oracle(p):
    for n in (0, 1, 2, 7, 64, 65, 1000, 262145):
        assert P.chunk_partition(n, p) == OC.chunk_partition(n, p)
        assert P.layout("ring", n, p) == OC.layout("ring", n, p)
        assert P.layout("rhd", n, p) == OC.layout("rhd", n, p)


@settings(max_examples=300, deadline=None)
@given(st.integers(0, 3_000_000), st.integers(1, 16), st.sampled_from([0, 1]), st.integers(1, 40))
def test_layout_pieces_cover_every_segment(n, p, layout, K):
    """cm_layout_piece (the host-gradient pipeline's unit, cm.h host_split):
    for every rank, the K pieces of its segment are consecutive, disjoint,
    cover the segment exactly and are cut on 64-element boundaries — so every
    element is reduced by the owner (and in the fold order) it has in the
    whole-buffer allreduce."""
    import ctypes as C
    whole = P.layout("ring" if layout == 0 else "rhd", n, p)
    off, ln = (C.c_int64 * p)(), (C.c_int64 * p)()
    for q, (o, l) in enumerate(whole):
        pos = o
        for k in range(K):
            assert L.lib.cm_layout_piece(layout, n, p, k, K, off, ln) == 0
            assert off[q] == pos and ln[q] >= 0
            if 0 < k:
                assert off[q] % 64 == 0 or off[q] in (o, o + l)
            pos += ln[q]
        assert pos == o + l
    assert L.lib.cm_layout_piece(layout, n, p, K, K, off, ln) != 0


@settings(max_examples=200, deadline=None)
@given(st.integers(0, 1000), st.integers(1, 64))
def test_chunk_partition_property(n, p):
    # test_core.py:112-125 invariants
    chunks = P.chunk_partition(n, p)
    assert len(chunks) == p
    assert sum(ln for _, ln in chunks) == n
    assert max(ln for _, ln in chunks) - min(ln for _, ln in chunks) <= 1
    off = 0
    for o, ln in chunks:
        assert o == off
        off += ln


def test_chunk_partition_errors():
    with pytest.raises(P.InvalidGroupError):
        P.chunk_partition(4, 0)
    with pytest.raises(P.ShapeError):
        P.chunk_partition(-1, 2)


def test_resolve_algorithm_reference_cases():
    # test_collectives.py:154-171
    assert P.resolve_algorithm("auto", 1024) == "rhd_rsa"
    assert P.resolve_algorithm("auto", 1 << 20) == "ring_rsa"
    assert P.resolve_algorithm("auto", P.DEFAULT_SWITCH_BYTES) == "ring_rsa"
    assert P.resolve_algorithm("auto", P.DEFAULT_SWITCH_BYTES - 1) == "rhd_rsa"
    for a in ("flat", "ring_rsa", "rhd_rsa"):
        assert P.resolve_algorithm(a, 1) == a
    with pytest.raises(P.ConfigError):
        P.resolve_algorithm("tree", 64)
    with pytest.raises(P.ConfigError):
        P.resolve_algorithm("auto", 64, switch_bytes=0)


def test_stats_match_golden_for_every_case():
    for case in of_kind("allreduce"):
        for r in range(case["p"]):
            got = P.algo_stats(case["algo"], case["p"], r, case["n"], case["dtype"])
            assert [got.rounds, got.messages_per_rank, got.bytes_sent_per_rank] == case["stats"][r], case


@pytest.mark.parametrize("layout", ["ring", "rhd"])
def test_rs_ag_stats_match_oracle(layout):
    for p in range(1, 10):
        for n in (0, 1, 7, 64, 1000):
            for r in range(p):
                s = L.Stats()
                L.check(L.lib.cm_rs_stats(L.LAYOUT[layout], p, r, n, L.DTYPE["float32"], L.C.byref(s)))
                assert (s.rounds, s.messages_per_rank, s.bytes_sent_per_rank) == \
                    OC.reduce_scatter_stats(layout, p, n, "float32", r)
                L.check(L.lib.cm_ag_stats(L.LAYOUT[layout], p, r, n, L.DTYPE["float32"], L.C.byref(s)))
                assert (s.rounds, s.messages_per_rank, s.bytes_sent_per_rank) == \
                    OC.allgather_stats(layout, p, n, "float32", r)
                # RS + AG = the whole allreduce schedule's messages and bytes
                full = OC.stats("ring_rsa" if layout == "ring" else "rhd_rsa", p, n, "float32", r)
                rs = OC.reduce_scatter_stats(layout, p, n, "float32", r)
                ag = OC.allgather_stats(layout, p, n, "float32", r)
                assert rs[1] + ag[1] == full[1] and rs[2] + ag[2] == full[2]


def _tensors(byte_sizes):
    return [P.Tensor(f"t{i}", "float32", np.arange(b // 4, dtype=np.float32))
            for i, b in enumerate(byte_sizes)]


def test_fuse_plan_reference_examples():
    # test_aggregation.py:71-92
    cfg = P.FusionConfig
    assert P.fuse_plan(_tensors([16, 16, 48, 128]), cfg(64)) == [[0, 1], [2], [3]]
    assert P.fuse_plan(_tensors([16, 16, 48, 128]), cfg(2 ** 40)) == [[0, 1, 2, 3]]
    assert P.fuse_plan(_tensors([16, 16, 48]), cfg(1)) == [[0], [1], [2]]
    mixed = [P.Tensor("a", "float32", np.zeros(2, np.float32)), P.Tensor("b", "float64", np.zeros(2))]
    assert len(P.fuse_plan(mixed, cfg(2 ** 20))) == 2


@settings(max_examples=100, deadline=None)
@given(st.lists(st.integers(1, 64), min_size=1, max_size=30), st.integers(1, 512))
def test_fuse_plan_matches_oracle_and_invariants(elem_counts, threshold):
    ts = [P.Tensor(f"t{i:02d}", "float32", np.ones(n, np.float32)) for i, n in enumerate(elem_counts)]
    plan = P.fuse_plan(ts, P.FusionConfig(threshold))
    assert plan == OA.fuse_plan([(t.name, t.dtype, t.nbytes) for t in ts], threshold)
    assert [i for g in plan for i in g] == list(range(len(ts)))
    for g in plan:
        if len(g) > 1:
            assert sum(ts[i].nbytes for i in g) <= threshold
    assert len(P.fuse_plan(ts, P.FusionConfig(threshold * 2))) <= len(plan)


def test_fuse_of_host_tensors_has_no_cpu_fallback():
    """fuse() puts the fused buffer on the GPU (CUDA-aware semantics; the
    GPU test checks the values): without a device it fails loudly instead
    of concatenating on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: covered by tests/test_gpu_fused_virtual.py")
    with pytest.raises((RuntimeError, AssertionError)):
        P.fuse(_tensors([16, 48, 32]), P.FusionConfig(2 ** 20))


REG = of_kind("registry")


@pytest.mark.parametrize("case", REG, ids=[f"{c['trace']}-{c['policy']}" for c in REG])
def test_sim_registry_replays_golden_traces(case):
    trace = dict(I.registry_traces())[case["trace"]]
    reg = P.BufferRegistry(case["policy"])
    handles, answers = {}, []
    for op in trace:
        try:
            if op[0] == "alloc":
                handles[op[1]] = reg.alloc(P.BufferKind(op[2]), op[3])
            elif op[0] == "free":
                reg.free(handles[op[1]])
            else:
                answers.append(reg.classify(handles[op[1]]).value)
        except P.CollectiumError as exc:
            answers.append(type(exc).__name__)
    assert answers == case["answers"]
    assert reg.stats_dict() == case["stats"]
    assert json.loads(reg.stats_json()) == case["stats"]
    assert {str(k): h.address for k, h in handles.items()} == case["addresses"]


def test_registry_reference_behaviours():
    # test_registry.py:11-120
    reg = P.BufferRegistry(P.Policy.INTERCEPT_CACHE)
    h1 = reg.alloc(P.BufferKind.DEVICE, 256)
    assert reg.stats.inserts == 1 and reg.classify(h1) is P.BufferKind.DEVICE
    assert reg.stats.driver_queries == 0
    reg = P.BufferRegistry(P.Policy.NO_CACHE)
    h1 = reg.alloc(P.BufferKind.DEVICE, 256)
    reg.free(h1)
    h2 = reg.alloc(P.BufferKind.HOST, 64)
    assert h2.address == h1.address
    with pytest.raises(P.InvalidHandleError):
        reg.free(h1)          # stale handle object: double free
    with pytest.raises(ValueError):
        reg.alloc(P.BufferKind.HOST, 0)
    for pol in P.Policy:
        with pytest.raises(P.UnknownBufferError):
            P.BufferRegistry(pol).classify(P.BufferHandle(0xDEAD, 8))
    reg = P.BufferRegistry(P.Policy.NO_CACHE, query_delay_ns=2000)
    h = reg.alloc(P.BufferKind.HOST, 8)
    reg.classify(h)
    reg.classify(h)
    assert reg.query_delay_seconds() == pytest.approx(4e-6)
    lazy = P.BufferRegistry(P.Policy.LAZY_CACHE)
    a = lazy.alloc(P.BufferKind.HOST, 32)
    assert lazy.classify(a) is P.BufferKind.HOST
    lazy.free(a)
    b = lazy.alloc(P.BufferKind.DEVICE, 32)
    assert lazy.classify(b) is P.BufferKind.HOST          # stale (PAPER §V-B)
    assert lazy.ground_truth(b) is P.BufferKind.DEVICE


@settings(max_examples=60, deadline=None)
@given(st.integers(0, 10_000), st.integers(10, 120))
def test_sim_registry_matches_oracle_on_random_traces(seed, length):
    trace = I.random_trace(seed, length)
    for pol in ("no_cache", "lazy_cache", "intercept_cache"):
        want_answers, want_stats, _ = OR.replay(trace, pol)
        reg = P.BufferRegistry(pol)
        handles, answers = {}, []
        for op in trace:
            try:
                if op[0] == "alloc":
                    handles[op[1]] = reg.alloc(P.BufferKind(op[2]), op[3])
                elif op[0] == "free":
                    reg.free(handles[op[1]])
                else:
                    answers.append(reg.classify(handles[op[1]]).value)
            except P.CollectiumError as exc:
                answers.append(type(exc).__name__)
        assert answers == want_answers
        assert reg.stats_dict() == {"policy": pol, **want_stats}
