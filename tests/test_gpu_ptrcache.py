"""The pointer cache on real memory (reference registry.py:52-151; PAPER §V-B).

``BufferRegistry(backend="cuda")``: allocations are real (cudaMalloc /
cudaHostAlloc), the driver query is one cuPointerGetAttributes (memory type,
device ordinal, allocation range, buffer id), and the intercept cache answers
interior pointers of registered ranges (torch sub-allocations). The counters
follow the reference semantics: no_cache queries on every classify,
lazy_cache once per address and never invalidates (stale after free),
intercept_cache never queries and rejects unknown addresses.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1810_11112_b200 as P  # noqa: E402

DEV, HOST = P.BufferKind.DEVICE, P.BufferKind.HOST


@pytest.mark.parametrize("policy", ["no_cache", "lazy_cache"])
def test_driver_backed_classification(policy):
    reg = P.BufferRegistry(policy, backend="cuda")
    d = reg.alloc(DEV, 1 << 20)
    h = reg.alloc(HOST, 4096)
    pageable = np.zeros(1000, np.float32)
    t = torch.empty(4096, device="cuda")
    sub = t[1000:]                                    # interior pointer of a torch block
    pin = torch.empty(4096).pin_memory()
    cases = [(d.address, DEV), (h.address, HOST), (pageable.ctypes.data, HOST),
             (sub.data_ptr(), DEV), (pin.data_ptr(), HOST)]
    for _ in range(3):
        for addr, kind in cases:
            assert reg.classify(addr) == kind
    st = reg.stats
    if policy == "no_cache":
        assert st.driver_queries == 3 * len(cases) and st.cache_hits == 0
    else:
        assert st.driver_queries == len(cases) and st.cache_hits == 2 * len(cases)
        assert st.inserts == len(cases)
    assert reg.query_delay_seconds() > 0             # measured wall time of the real queries
    info = reg.info(d)
    assert info["kind"] == DEV and info["device"] == torch.cuda.current_device()
    assert info["range_start"] == d.address and info["range_size"] >= 1 << 20 and info["buffer_id"] > 0
    si = reg.info(sub.data_ptr())
    assert si["range_start"] <= sub.data_ptr() < si["range_start"] + si["range_size"]
    assert si["buffer_id"] == reg.info(t.data_ptr())["buffer_id"]   # same allocation
    assert reg.info(pageable.ctypes.data)["device"] == -1
    reg.free(d)
    reg.free(h)


def test_lazy_cache_is_stale_after_free_intercept_is_not():
    lazy = P.BufferRegistry("lazy_cache", backend="cuda")
    d = lazy.alloc(DEV, 1 << 16)
    addr = d.address
    assert lazy.classify(addr) == DEV
    q = lazy.stats.driver_queries
    lazy.free(d)
    # registry.py:101-102: the lazy entry is never invalidated — still DEVICE,
    # no new query, although the driver no longer knows the address as device memory
    assert lazy.classify(addr) == DEV and lazy.stats.driver_queries == q
    assert lazy.stats.invalidations == 0
    ic = P.BufferRegistry("intercept_cache", backend="cuda")
    d = ic.alloc(DEV, 1 << 16)
    assert ic.classify(d) == DEV and ic.stats.driver_queries == 0
    ic.free(d)
    assert ic.stats.invalidations == 1
    with pytest.raises(P.UnknownBufferError):
        ic.classify(d.address)


def test_intercept_cache_range_map_for_torch_sub_allocations():
    reg = P.BufferRegistry("intercept_cache", backend="cuda")
    t = torch.empty(1 << 20, device="cuda")
    with pytest.raises(P.UnknownBufferError):
        reg.classify(t.data_ptr())
    reg.register(t.data_ptr(), t.numel() * 4, DEV)
    for off in (0, 1, 12345, (1 << 20) - 1):
        assert reg.classify(t[off:].data_ptr()) == DEV          # interior pointers
    with pytest.raises(P.UnknownBufferError):
        reg.classify(t.data_ptr() + t.numel() * 4)             # one past the end
    info = reg.info(t[777:].data_ptr())
    assert info["range_start"] == t.data_ptr() and info["range_size"] == t.numel() * 4
    assert reg.stats.driver_queries == 0
    reg.unregister(t.data_ptr())
    with pytest.raises(P.UnknownBufferError):
        reg.classify(t[5:].data_ptr())
    assert reg.stats.invalidations == 1
