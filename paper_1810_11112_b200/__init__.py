"""B200-native CUDA-aware allreduce (arXiv 1810.11112) with the reference
``collectium`` API surface for the allreduce hot path: size-threshold
algorithm selection, recursive halving/doubling and ring reduce-scatter +
allgather replayed bit-exactly by sm_100a kernels over CUDA-IPC NVLink peer
memory, tensor fusion of gradient buffers, and the pointer cache.

Importing requires the built ``libcm.so`` (no CPU fallback).
"""

from .errors import (CollectiumError, ConfigError, DeadlockError,  # noqa: F401
                     InvalidGroupError, InvalidHandleError, ProtocolError,
                     RoutingError, ShapeError, StalledProducerError,
                     TransportError, UnknownBufferError,
                     UnsupportedOperationError)
from .core import (DTYPES, GroupSpec, ReduceOp, Tensor, chunk_partition,  # noqa: F401
                   layout, local_reduce)
from .comm import Communicator, VirtualGroup  # noqa: F401
from .collectives import (ALGORITHMS, DEFAULT_SWITCH_BYTES, CollectiveStats,  # noqa: F401
                          algo_stats, allgather, allgather_group, allreduce,
                          allreduce_flat, allreduce_group, allreduce_rhd,
                          allreduce_ring, reduce_scatter, reduce_scatter_group,
                          resolve_algorithm)
from .aggregation import (DEFAULT_FUSION_THRESHOLD, FusedBuffer, FusionConfig,  # noqa: F401
                          GradientSet, aggregate, aggregate_group, fuse,
                          negotiate_ready_group, register_gradients_group,
                          fuse_plan, negotiate_ready, register_gradients, unfuse)
from .overlap import OverlappedAggregator  # noqa: F401
from .paramserver import PsTopology, run_ps_step, run_ps_step_group  # noqa: F401
from .registry import (BufferHandle, BufferKind, BufferRegistry, Policy,  # noqa: F401
                       RegistryStats)

__version__ = "0.1.0"
