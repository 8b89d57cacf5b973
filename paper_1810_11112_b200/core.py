"""Value types of the allreduce path: Tensor, ReduceOp, GroupSpec,
local_reduce, chunk_partition (reference core.py:18-130).

``Tensor.payload`` is a 1-D contiguous torch tensor, on a CUDA device (the
normal case) or in host memory (CUDA-aware semantics: host buffers are
staged through the device by the communicator). numpy arrays and lists are
accepted and become host tensors.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .errors import InvalidGroupError, ShapeError

# core.py:18-21 pins float32/float64; bfloat16 and int32/int64 are extensions
DTYPES = {
    "float32": torch.float32,
    "float64": torch.float64,
    "bfloat16": torch.bfloat16,
    "int32": torch.int32,
    "int64": torch.int64,
}
_NP_STORE = {"float32": np.dtype("<f4"), "float64": np.dtype("<f8"),
             "bfloat16": np.dtype("<u2"), "int32": np.dtype("<i4"), "int64": np.dtype("<i8")}
_TORCH_NAME = {v: k for k, v in DTYPES.items()}


class ReduceOp(enum.Enum):
    """core.py:24-26."""
    SUM = "sum"
    MAX = "max"


def _as_payload(values, dtype: str) -> torch.Tensor:
    if type(values) is torch.Tensor and values.dtype == DTYPES[dtype] and values.dim() == 1 \
            and values.is_contiguous():
        return values                                  # fast path: already a 1-D payload
    if isinstance(values, torch.Tensor):
        t = values
        if t.dtype != DTYPES[dtype]:
            t = t.to(DTYPES[dtype])
    else:
        arr = np.asarray(values)
        if dtype == "bfloat16":
            if arr.dtype == np.uint16:
                t = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1).copy()).view(torch.bfloat16)
            else:
                t = torch.as_tensor(np.asarray(arr, dtype=np.float32)).to(torch.bfloat16)
        else:
            t = torch.from_numpy(np.ascontiguousarray(arr, dtype=_NP_STORE[dtype]).copy())
    return t.reshape(-1).contiguous()


@dataclass(frozen=True)
class Tensor:
    """Named, contiguous 1-D payload; the unit of reduction (core.py:29-70)."""

    name: str
    dtype: str
    payload: torch.Tensor

    def __post_init__(self):
        if self.dtype not in DTYPES:
            raise ShapeError(f"unsupported dtype {self.dtype!r}")
        object.__setattr__(self, "payload", _as_payload(self.payload, self.dtype))

    @classmethod
    def _wrap(cls, name: str, dtype: str, payload: torch.Tensor) -> "Tensor":
        """Internal constructor for payloads the library produced itself
        (already 1-D, contiguous, right dtype): skips validation."""
        t = object.__new__(cls)
        object.__setattr__(t, "name", name)
        object.__setattr__(t, "dtype", dtype)
        object.__setattr__(t, "payload", payload)
        return t

    @property
    def len(self) -> int:
        return int(self.payload.shape[0])

    @property
    def nbytes(self) -> int:
        return int(self.payload.numel() * self.payload.element_size())

    @property
    def is_cuda(self) -> bool:
        return self.payload.is_cuda

    def to_bytes(self) -> bytes:
        """Little-endian element bytes (bfloat16: raw 16-bit patterns)."""
        t = self.payload.detach()
        if t.is_cuda:
            t = t.cpu()
        if self.dtype == "bfloat16":
            t = t.view(torch.int16)
        return t.numpy().tobytes()

    def numpy(self) -> np.ndarray:
        return np.frombuffer(self.to_bytes(), dtype=_NP_STORE[self.dtype]).copy()

    @classmethod
    def from_bytes(cls, name: str, dtype: str, raw: bytes) -> "Tensor":
        if dtype not in DTYPES:
            raise ShapeError(f"unsupported dtype {dtype!r}")
        itemsize = _NP_STORE[dtype].itemsize
        if len(raw) % itemsize:
            raise ShapeError(f"payload of {len(raw)} bytes is not a whole number of {dtype} elements")
        return cls(name, dtype, np.frombuffer(raw, dtype=_NP_STORE[dtype]))

    def with_payload(self, values) -> "Tensor":
        return Tensor(self.name, self.dtype, values)


@dataclass(frozen=True)
class GroupSpec:
    """A process group of ``size`` ranks numbered densely 0..size-1 (core.py:73-91)."""

    size: int

    def __post_init__(self):
        if self.size < 1:
            raise InvalidGroupError(f"group size must be >= 1, got {self.size}")

    @property
    def ranks(self) -> range:
        return range(self.size)

    def check_rank(self, rank: int) -> None:
        if not 0 <= rank < self.size:
            raise InvalidGroupError(f"rank {rank} outside group of size {self.size}")


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def local_reduce(a: Tensor, b: Tensor, op: ReduceOp) -> Tensor:
    """Element-wise ``a op b`` with ``a`` as the accumulator (core.py:94-110),
    computed by the sm_100a kernel ``cm_local_reduce``. Host payloads are
    staged to the current CUDA device and the result is returned on the host."""
    if a.len != b.len:
        raise ShapeError(f"length mismatch: {a.len} vs {b.len}")
    if a.dtype != b.dtype:
        raise ShapeError(f"dtype mismatch: {a.dtype} vs {b.dtype}")
    dev = a.payload.device if a.is_cuda else (b.payload.device if b.is_cuda else
                                              torch.device("cuda", torch.cuda.current_device()))
    x = a.payload.to(dev, non_blocking=True)
    y = b.payload.to(dev, non_blocking=True)
    out = torch.empty_like(x)
    with torch.cuda.device(dev):
        L.check(L.lib.cm_local_reduce(x.data_ptr(), y.data_ptr(), out.data_ptr(), a.len,
                                      L.DTYPE[a.dtype], L.OP[op.value], _stream_ptr(dev)))
    if not a.is_cuda:
        out = out.cpu()
    return Tensor(a.name, a.dtype, out)


def chunk_partition(n: int, p: int) -> list[tuple[int, int]]:
    """p contiguous chunks, the first ``n mod p`` one element longer
    (core.py:113-130); computed by the C library (cm_chunk_partition)."""
    if p < 1:
        raise InvalidGroupError(f"cannot partition over p={p} processes")
    if n < 0:
        raise ShapeError(f"negative element count {n}")
    off = (L.C.c_int64 * p)()
    ln = (L.C.c_int64 * p)()
    L.check(L.lib.cm_chunk_partition(n, p, off, ln))
    return [(int(off[i]), int(ln[i])) for i in range(p)]


def layout(kind: str, n: int, p: int) -> list[tuple[int, int]]:
    """Per-rank (offset, length) owned after a reduce-scatter: "ring" is
    chunk_partition, "rhd" the recursive-halving segments (folded odd ranks
    own nothing)."""
    if kind not in L.LAYOUT:
        from .errors import ConfigError
        raise ConfigError(f"unknown layout {kind!r}")
    off = (L.C.c_int64 * p)()
    ln = (L.C.c_int64 * p)()
    L.check(L.lib.cm_layout(L.LAYOUT[kind], n, p, off, ln))
    return [(int(off[i]), int(ln[i])) for i in range(p)]
