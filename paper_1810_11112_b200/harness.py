"""Benchmark harness with the reference's flags, CSV and exit codes.

Restates ``collectium.bench`` (pkg/src/collectium/bench.py) for the NVLink
communicator so results can be emitted in the reference's own format:

* ``microbench`` (bench.py:176-219): osu-style allreduce latency sweep over
  powers of two from ``msg_min_bytes`` to ``msg_max_bytes``; float64 payload
  of ``size // 8`` elements seeded ``default_rng([seed, size, rank])``;
  per-iteration host wall time of one blocking allreduce, element-wise max
  over ranks, mean/min/max on rank 0 (bench.py:142-167). CSV header
  ``MICROBENCH_CSV_HEADER`` (bench.py:38-39) followed by three extra
  columns: ``device_latency_s`` (CUDA events, max over ranks), ``bus_gbps``
  (nccl-tests convention) and ``roofline_frac`` (busBW / 770 GB/s measured
  NVLink peer copy).
* ``train`` (bench.py:235-284): synthetic gradients per (seed, iteration,
  layer, rank) (bench.py:224-232), the modeled forward+backward time spent
  for real as the socket transport does (sockets.py:206-210, a sleep), then
  ``aggregate`` (``horovod_allreduce`` with ``algo``, ``baidu_ring`` with
  ring_rsa) or the parameter-server step (``ps_pull``, paramserver.py via
  ``run_ps_step``). CSV ``TRAIN_CSV_HEADER`` (bench.py:40).

* ``sweep`` (bench.py:287-291): the analytic alpha-beta-gamma model
  (costmodel.py, a restatement of simcost.py), with the reference's default
  costs, a JSON cost model, or ``--cost-model b200`` (fitted to this
  framework's measured latencies).

Group identity comes from torchrun's ``RANK``/``WORLD_SIZE`` or the
reference's ``COLLECTIUM_RANK``/``COLLECTIUM_NPROCS`` (bench.py:32-33,
316-334). The simulator and socket transport are not part of this framework
(DESIGN.md section 7): asking for them is a ``ConfigError`` (exit 2).
"""

from __future__ import annotations

import json
import os
import time
from dataclasses import dataclass, field, fields

import numpy as np

from .aggregation import DEFAULT_FUSION_THRESHOLD, FusionConfig, GradientSet, aggregate
from .collectives import ALGORITHMS, DEFAULT_SWITCH_BYTES, ReduceOp, allreduce, algo_stats, resolve_algorithm
from .core import GroupSpec, Tensor
from .errors import ConfigError

ENV_NPROCS = "COLLECTIUM_NPROCS"
ENV_RANK = "COLLECTIUM_RANK"
MICROBENCH_CSV_HEADER = ("message_bytes,algo,p,mean_latency_s,min_latency_s,"
                         "max_latency_s,messages_per_rank")
MICROBENCH_EXTRA = "device_latency_s,bus_gbps,roofline_frac"
TRAIN_CSV_HEADER = "model,strategy,p,images_per_sec,ideal,efficiency"
NVLINK_PEAK_GBS = 770.0
STRATEGIES = ("horovod_allreduce", "baidu_ring", "ps_pull")
_MODES = ("microbench", "train", "sweep")
_TRANSPORTS = ("nvlink", "sim", "socket")


@dataclass(frozen=True)
class ModelSpec:
    """simcost.py ModelSpec: per-layer (gradient bytes, backward seconds)."""
    name: str
    layers: tuple
    forward_s: float
    batch_size: int = 64

    @property
    def backward_s(self) -> float:
        return sum(s for _, s in self.layers)

    @classmethod
    def from_dict(cls, data: dict) -> "ModelSpec":
        try:
            return cls(name=str(data["name"]),
                       layers=tuple((int(b), float(s)) for b, s in data["layers"]),
                       forward_s=float(data["forward_s"]),
                       batch_size=int(data.get("batch_size", 64)))
        except (KeyError, TypeError, ValueError) as exc:
            raise ConfigError(f"malformed model spec: {exc}") from exc


def _uniform(name, n_layers, layer_bytes, backward_s, forward_s) -> ModelSpec:
    return ModelSpec(name, tuple((layer_bytes, backward_s / n_layers) for _ in range(n_layers)), forward_s)


def builtin_models() -> dict:
    """simcost.py:152-163 (the reference's calibration artifacts)."""
    return {
        "mobilenet_like": _uniform("mobilenet_like", 28, 600_000, 0.0114, 0.0057),
        "resnet50_like": _uniform("resnet50_like", 53, 1_920_000, 0.524, 0.262),
        "nasnet_like": _uniform("nasnet_like", 60, 5_880_000, 1.855, 0.927),
    }


def resolve_model(name_or_path: str) -> ModelSpec:
    models = builtin_models()
    if name_or_path in models:
        return models[name_or_path]
    try:
        with open(name_or_path, encoding="utf-8") as fh:
            return ModelSpec.from_dict(json.load(fh))
    except OSError as exc:
        raise ConfigError(f"model {name_or_path!r} is neither a built-in ({sorted(models)}) "
                          f"nor a readable spec file") from exc


@dataclass
class BenchConfig:
    """bench.py:44-104 BenchConfig (same fields and validation; transport
    "nvlink" is this framework's communicator and the default)."""
    mode: str = "microbench"
    transport: str = "nvlink"
    algo: str = "auto"
    switch_bytes: int = DEFAULT_SWITCH_BYTES
    fusion_threshold: int = DEFAULT_FUSION_THRESHOLD
    strategy: str = "horovod_allreduce"
    model: str = "resnet50_like"
    p: int = 1
    warmup_iters: int = 5
    timed_iters: int = 10
    seed: int = 0
    output: str | None = None
    hostfile: str | None = None
    rank: int | None = None
    msg_min_bytes: int = 8
    msg_max_bytes: int = 268435456
    recv_timeout: float = 30.0
    rendezvous_timeout: float = 30.0
    learning_rate: float = 0.1
    models: list = field(default_factory=lambda: ["mobilenet_like", "resnet50_like", "nasnet_like"])
    strategies: list = field(default_factory=lambda: list(STRATEGIES))
    p_list: list = field(default_factory=lambda: [1, 2, 4, 8])
    dump_grads: str | None = None
    cost_model: object = None          # CostModel, or "b200" (measured calibration per p)

    def validate(self) -> None:
        if self.mode not in _MODES:
            raise ConfigError(f"mode must be one of {_MODES}, got {self.mode!r}")
        if self.transport not in _TRANSPORTS:
            raise ConfigError(f"transport must be one of {_TRANSPORTS}, got {self.transport!r}")
        if self.algo not in ALGORITHMS:
            raise ConfigError(f"algo must be one of {ALGORITHMS}")
        if self.strategy not in STRATEGIES:
            raise ConfigError(f"strategy must be one of {STRATEGIES}")
        if self.timed_iters < 1:
            raise ConfigError("timed_iters must be >= 1")
        if self.warmup_iters < 0:
            raise ConfigError("warmup_iters must be >= 0")
        if self.p < 1:
            raise ConfigError("p must be >= 1")
        if self.switch_bytes <= 0:
            raise ConfigError("switch_bytes must be > 0")
        if self.fusion_threshold <= 0:
            raise ConfigError("fusion_threshold must be > 0")
        if self.msg_min_bytes < 8 or self.msg_min_bytes % 8:
            raise ConfigError("msg_min_bytes must be a multiple of 8, >= 8")
        if self.msg_max_bytes < self.msg_min_bytes:
            raise ConfigError("msg_max_bytes must be >= msg_min_bytes")
        if self.mode == "sweep":            # analytic: no transport involved
            return
        if self.transport != "nvlink":
            raise ConfigError(f"transport {self.transport!r} (the reference's simulator / TCP "
                              f"sockets) is not part of this framework; use transport 'nvlink'")

    @classmethod
    def from_file(cls, path: str) -> "BenchConfig":
        try:
            with open(path, encoding="utf-8") as fh:
                data = json.load(fh)
        except OSError as exc:
            raise ConfigError(f"cannot read config {path}: {exc}") from exc
        except json.JSONDecodeError as exc:
            raise ConfigError(f"{path}:{exc.lineno}: invalid JSON: {exc.msg}") from exc
        known = {f.name for f in fields(cls)}
        unknown = set(data) - known
        if unknown:
            raise ConfigError(f"{path}: unknown fields {sorted(unknown)}")
        if isinstance(data.get("cost_model"), dict):
            from .costmodel import CostModel
            data = dict(data, cost_model=CostModel.from_dict(data["cost_model"]))
        try:
            return cls(**data)
        except TypeError as exc:
            raise ConfigError(f"{path}: {exc}") from exc


def message_sizes(cfg: BenchConfig) -> list:
    sizes, size = [], cfg.msg_min_bytes
    while size <= cfg.msg_max_bytes:
        sizes.append(size)
        size *= 2
    return sizes


def fmt(x: float) -> str:
    """bench.py:170-171: 9 significant digits."""
    return format(x, ".9g")


def resolve_identity(cfg: BenchConfig) -> tuple:
    """(rank, size): torchrun's RANK/WORLD_SIZE, else --rank /
    COLLECTIUM_RANK with COLLECTIUM_NPROCS (bench.py:316-334), else (0, 1)."""
    env_np = os.environ.get("WORLD_SIZE") or os.environ.get(ENV_NPROCS)
    size = int(env_np) if env_np is not None else 1
    rank = cfg.rank
    if rank is None:
        env_rank = os.environ.get("RANK") or os.environ.get(ENV_RANK)
        rank = int(env_rank) if env_rank is not None else 0
    if not 0 <= rank < size:
        raise ConfigError(f"rank {rank} outside a group of {size} ranks")
    return rank, size


class _Group:
    """Bootstraps torch.distributed (host control plane, gloo) and the NVLink
    communicator for this process's rank."""

    def __init__(self, cfg: BenchConfig, staging_bytes: int):
        import torch
        import torch.distributed as dist
        from .comm import Communicator
        self.rank, self.size = resolve_identity(cfg)
        self.local = int(os.environ.get("LOCAL_RANK", self.rank)) % max(1, torch.cuda.device_count())
        torch.cuda.set_device(self.local)
        self.own_pg = False
        if self.size > 1 and not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            dist.init_process_group("gloo", rank=self.rank, world_size=self.size)
            self.own_pg = True
        self.comm = Communicator(self.rank, self.size, self.local, staging_bytes=staging_bytes,
                                 pool_bytes=2 << 20, timeout_s=cfg.recv_timeout)
        self.group = GroupSpec(self.size)

    def max_over_ranks(self, values: list) -> list:
        import torch
        import torch.distributed as dist
        t = torch.tensor(values, dtype=torch.float64)
        if self.size > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def close(self):
        import torch.distributed as dist
        self.comm.close()
        if self.own_pg:
            dist.destroy_process_group()


def run_microbench(cfg: BenchConfig) -> list:
    """bench.py:176-219 on the NVLink communicator; returns CSV rows."""
    import torch
    cfg.validate()
    g = _Group(cfg, staging_bytes=max(64 << 20, 2 * cfg.msg_max_bytes))
    rows = [MICROBENCH_CSV_HEADER + "," + MICROBENCH_EXTRA]
    try:
        for size in message_sizes(cfg):
            count = size // 8
            rng = np.random.default_rng([cfg.seed, size, g.rank])
            x = torch.from_numpy(rng.standard_normal(count)).cuda()
            t = Tensor("payload", "float64", x)
            algo = resolve_algorithm(cfg.algo, size, cfg.switch_bytes)
            out = torch.empty_like(x)
            times, dev, messages = [], [], None
            g.comm.blocking = False
            for it in range(cfg.warmup_iters + cfg.timed_iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0 = time.perf_counter()
                e0.record()
                _, stats = allreduce(t, ReduceOp.SUM, g.group, g.comm, algo=algo, out=out)
                e1.record()
                g.comm.synchronize()           # blocking semantics of the reference call
                t1 = time.perf_counter()
                if it >= cfg.warmup_iters:
                    times.append(t1 - t0)
                    e1.synchronize()
                    dev.append(e0.elapsed_time(e1) * 1e-3)
                    messages = stats.messages_per_rank
            worst = g.max_over_ranks(times)
            dworst = g.max_over_ranks(dev)
            mean, dmean = sum(worst) / len(worst), sum(dworst) / len(dworst)
            p = g.size
            bus = size * 2 * (p - 1) / p / dmean / 1e9 if p > 1 else 0.0
            rows.append(",".join([str(size), algo, str(p), fmt(mean), fmt(min(worst)), fmt(max(worst)),
                                  str(messages), fmt(dmean), fmt(bus), fmt(bus / NVLINK_PEAK_GBS)]))
    finally:
        g.close()
    return rows


def synth_gradients(seed: int, iteration: int, model: ModelSpec, rank: int, device) -> GradientSet:
    """bench.py:224-232: float32 standard normal per (seed, iteration, layer, rank)."""
    import torch
    ts = []
    for idx, (nbytes, _) in enumerate(model.layers):
        rng = np.random.default_rng([seed, iteration, idx, rank])
        a = rng.standard_normal(nbytes // 4, dtype=np.float32)
        ts.append(Tensor(f"layer{idx:04d}", "float32", torch.from_numpy(a).to(device)))
    return GradientSet(tuple(ts), iteration)


def run_train_bench(cfg: BenchConfig) -> tuple:
    """bench.py:235-284 (horovod_allreduce / baidu_ring) on the NVLink
    communicator; returns (CSV rows, final tensors)."""
    import torch
    cfg.validate()
    model = resolve_model(cfg.model)
    grad_bytes = sum(b for b, _ in model.layers)
    ps = cfg.strategy == "ps_pull"
    need = 2 * grad_bytes if ps else min(grad_bytes, cfg.fusion_threshold)
    g = _Group(cfg, staging_bytes=max(64 << 20, need + (8 << 20)))
    try:
        fusion = FusionConfig(cfg.fusion_threshold)
        algo = "ring_rsa" if cfg.strategy == "baidu_ring" else cfg.algo
        device = torch.device("cuda", g.local)
        times, final = [], None
        if ps:                                   # bench.py:239-243: zero parameters, round-robin shards
            from .paramserver import PsTopology, run_ps_step
            names = [f"layer{idx:04d}" for idx in range(len(model.layers))]
            topology = PsTopology.create(range(g.size), range(g.size), names)
            params = [Tensor(nm, "float32", torch.zeros(nb // 4, dtype=torch.float32, device=device))
                      for nm, (nb, _) in zip(names, model.layers)]
        for it in range(cfg.warmup_iters + cfg.timed_iters):
            t0 = time.perf_counter()
            time.sleep(model.forward_s + model.backward_s)   # modeled compute (sockets.py:206-210)
            grads = synth_gradients(cfg.seed, it, model, g.rank, device)
            if ps:
                params = run_ps_step(g.rank, g.comm, topology, list(grads.tensors), params, cfg.learning_rate)
                final = params
            else:
                result = aggregate(grads, g.group, g.comm, algo=algo, cfg=fusion, switch_bytes=cfg.switch_bytes)
                final = list(result.tensors)
            t1 = time.perf_counter()
            if it >= cfg.warmup_iters:
                times.append(t1 - t0)
        worst = g.max_over_ranks(times)
        p = g.size
        ips = p * model.batch_size / (sum(worst) / len(worst))
        ideal = p * model.batch_size / (model.forward_s + model.backward_s)
        row = ",".join([model.name, cfg.strategy, str(p), fmt(ips), fmt(ideal), fmt(ips / ideal)])
        return [TRAIN_CSV_HEADER, row], final
    finally:
        g.close()


def write_output(cfg: BenchConfig, rows: list) -> None:
    text = "\n".join(rows) + "\n"
    if cfg.output:
        with open(cfg.output, "w", encoding="utf-8") as fh:
            fh.write(text)
    else:
        print(text, end="")


def run_sweep(cfg: BenchConfig) -> list:
    """bench.py:287-291 / simcost.py:265-290: analytic images/sec and
    scaling efficiency per (model, strategy, p); ``cost_model="b200"`` uses
    the alpha/beta/gamma fitted to this framework's measured latencies."""
    from .costmodel import CostModel, sweep, sweep_csv_rows
    cfg.validate()
    calibrated = cfg.cost_model == "b200"
    costs = cfg.cost_model if isinstance(cfg.cost_model, CostModel) else CostModel()
    return sweep_csv_rows(sweep(cfg.models, cfg.strategies, cfg.p_list, costs, cfg.fusion_threshold,
                                calibrated=calibrated))


def run_bench(cfg: BenchConfig) -> None:
    """bench.py:337-361."""
    cfg.validate()
    if cfg.mode == "sweep":
        write_output(cfg, run_sweep(cfg))
        return
    rank, _ = resolve_identity(cfg)
    if cfg.mode == "microbench":
        rows = run_microbench(cfg)
        if rank == 0:
            write_output(cfg, rows)
        return
    rows, final = run_train_bench(cfg)
    if rank == 0:
        write_output(cfg, rows)
    if cfg.dump_grads and rank == 0:      # results are identical on every rank
        np.savez(cfg.dump_grads, **{t.name: t.payload.cpu().numpy() for t in final})


__all__ = ["BenchConfig", "ModelSpec", "MICROBENCH_CSV_HEADER", "TRAIN_CSV_HEADER", "builtin_models",
           "resolve_model", "message_sizes", "run_microbench", "run_train_bench", "run_bench",
           "resolve_identity", "algo_stats"]
