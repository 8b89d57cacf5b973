#!/usr/bin/env python
"""Benchmark of the CUDA-aware allreduce hot path on B200.

Headline (default): BASELINE config 5 — the ResNet-50 gradient set
(resnet50_like: 53 x 480,000 fp32 = 25.44 M params, 101.76 MB per rank) run
through ``aggregate()`` every step: negotiation, tensor fusion under the
64 MB threshold (2 fused buffers), the NVLink allreduce with the fused mean.
One JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W]
    torchrun --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...   # the reference CPU path (threaded port)
    torchrun ... bench.py --mode sweep      # C2/C3 latency + busBW sweep vs NCCL (CSV)
    torchrun ... bench.py --mode tune       # measure the rhd/ring switch -> tuning.json

value   = N x 101.76 MB / device step time (GB/s of gradients aggregated,
          whole job); inputs resident in HBM, L2 flushed between steps.
e2e     = same metric through the public API with pinned HOST gradients
          (H2D + D2H inside the timed region).
roofline: N>=2 the collective kernel (busBW vs the measured 770 GB/s NVLink
          peer-copy rate); N=1 the fused pack kernel (HBM vs MEASURED_PEAKS).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "allreduce latency (us) and bus GB/s vs message size at 1/2/4/8 B200"
MODELS = {"resnet50_like": [480_000] * 53, "mobilenet_like": [150_000] * 28}
NVLINK_PEAK_GBS = 770.0      # B200_PROFILING.md: measured NVLink peer copy per direction
NVLINK_NOMINAL_GBS = 900.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


_RESULT_FD = None


def _isolate_stdout():
    """Route fd 1 (NCCL/torch banners, C-level prints) to stderr so stdout
    carries exactly the one JSON result line."""
    global _RESULT_FD
    if _RESULT_FD is None:
        sys.stdout.flush()
        _RESULT_FD = os.dup(1)
        os.dup2(2, 1)


def emit(obj) -> None:
    line = json.dumps(obj) + "\n"
    if _RESULT_FD is None:
        sys.stdout.write(line)
        sys.stdout.flush()
    else:
        os.write(_RESULT_FD, line.encode())


# --------------------------------------------------------------------------- env
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def init_dist(rank, world, local, nccl=True):
    if world == 1:
        return
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    backend = "cpu:gloo,cuda:nccl" if nccl else "gloo"
    kw = {"device_id": torch.device("cuda", local)} if nccl else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        dist.barrier()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons (NVML) every ~2 ms; the summary
    only uses samples taken inside the timed window (mark_start/mark_stop)."""

    def __init__(self, device_index: int):
        super().__init__(daemon=True)
        self.idx = device_index
        self.samples = []            # (t, mhz, reasons)
        self.stop_flag = threading.Event()
        self.ready = threading.Event()
        self.max_mhz = None
        self.t0 = self.t1 = None
        self.error = None

    def run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                     0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}
            self.ready.set()
            while not self.stop_flag.is_set():
                mhz = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((time.perf_counter(), mhz, [nm for bit, nm in names.items() if r & bit]))
                time.sleep(0.002)
        except Exception as exc:  # pragma: no cover
            self.error = f"nvml_unavailable:{type(exc).__name__}"
            self.ready.set()

    def start_and_wait(self):
        self.start()
        self.ready.wait(timeout=30)

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_stop(self):
        self.t1 = time.perf_counter()

    def result(self):
        self.stop_flag.set()
        self.join(timeout=2)
        win = [s for s in self.samples if self.t0 is not None and self.t0 <= s[0] <= (self.t1 or 1e30)]
        if not win and self.samples:     # very short timed window: nearest samples
            win = sorted(self.samples, key=lambda s: abs(s[0] - (self.t0 or 0)))[:3]
        reasons = sorted({r for s in win for r in s[2]} | ({self.error} if self.error else set()))
        med = statistics.median([s[1] for s in win]) if win else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "samples": len(win), "reasons": reasons}


# --------------------------------------------------------------------- workload
def make_grads(model, rank, device, dtype="float32", pinned=False):
    """Reference synth_gradients recipe (bench.py:224-232): default_rng([seed,
    it, layer, rank]).standard_normal(n, float32); bf16 = RNE of those."""
    import paper_1810_11112_b200 as P
    from tests.golden.inputs import synth_gradients
    ts = []
    grads = synth_gradients(0, 0, MODELS[model], rank)
    flat = None
    if device is None and pinned:     # host gradients: views of ONE flat pinned buffer, as a
        tdt = torch.bfloat16 if dtype == "bfloat16" else torch.float32   # framework's flat grads
        flat = torch.empty(sum(a.size for _, a in grads), dtype=tdt).pin_memory()
    off = 0
    for nm, a in grads:
        t = torch.from_numpy(a)
        if dtype == "bfloat16":
            t = t.to(torch.bfloat16)
        if device is not None:
            t = t.to(device)
        elif flat is not None:
            v = flat[off:off + a.size]
            v.copy_(t)
            t = v
            off += a.size
        ts.append(P.Tensor(nm, dtype, t))
    return P.GradientSet(tuple(ts))


def oracle_check(model, world, rank, res, dtype):
    """Rank 0: bit-exact comparison of this rank's aggregate with the CPU
    oracle (reference fold order) on the same synthetic inputs."""
    from oracle import aggregation as OA
    from oracle import collectives as OC
    from tests.golden.inputs import synth_gradients
    per_rank = [synth_gradients(0, 0, MODELS[model], r) for r in range(world)]
    if dtype == "bfloat16":
        per_rank = [[(nm, OC.f32_to_bf16(a)) for nm, a in g] for g in per_rank]
    want, _, _ = OA.aggregate(per_rank, dtype)
    for t in res.tensors:
        got = np.frombuffer(t.to_bytes(), dtype=OC.STORAGE[dtype])
        if not np.array_equal(got.view(np.uint8), np.asarray(want[t.name]).view(np.uint8)):
            return f"MISMATCH in {t.name}"
    return "bit-exact vs oracle (reference fold order)"


def cpu_baseline_sample(model, p, dtype="float32", max_s=20.0):
    """The reference path (threaded message-passing port of collectives.py /
    aggregation.py) on host cores, p ranks in-process."""
    from oracle import threaded as T
    from tests.golden.inputs import synth_gradients
    grads = [synth_gradients(0, 0, MODELS[model], r) for r in range(p)]
    times = []
    t_end = time.perf_counter() + max_s
    while True:
        t0 = time.perf_counter()
        T.ThreadNet(p).run(lambda r, tp: T.aggregate_rank(grads[r], tp))
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end or len(times) >= 3:
            break
    return times


# ----------------------------------------------------- virtual-group evidence
def virtual_block(args, local, steps):
    """N = 1 only: the reduction / allgather kernels the N >= 2 headline runs,
    driven as p virtual ranks on this GPU (one cooperative launch holds every
    rank's CTAs; flags, staging and fold order exactly as over NVLink).

    * C1 (BASELINE config 1): 4 ranks, 1 MiB fp32, auto (= ring_rsa), sum —
      device latency per call (L2-warm) and bit-exactness vs the reference
      golden SHA.
    * The headline kernel configuration (registered gradients, ONE
      multi-buffer two-shot launch with the fused mean) on the C5
      resnet50_like gradient set at p = 4 and p = 8: per-launch CUDA-event
      time of the collective kernel and its algorithmic HBM bytes. On one GPU
      every "peer" byte is an HBM byte. Algorithmic (compulsory) bytes: every
      rank's gradients read once and every rank's means written once, 2pS
      per launch. The kernel also moves each rank's reduced segment through
      staging (S/p written, (p-1)S/p read by the peers): 3pS moved, the
      staging part mostly L2-resident (ncu DRAM bytes in profiles/)."""
    import hashlib

    import paper_1810_11112_b200 as P
    from paper_1810_11112_b200 import _lib as L
    from tests.golden import inputs as I
    from tests.golden.load import of_kind
    device = torch.device("cuda", local)
    pk, pk_src = peaks()
    out = {"what": "p virtual ranks on this GPU (cooperative launch), the kernels of the N>=2 path",
           "peak": pk["hbm_gbs"], "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_src})"}

    def prof(vg, kind):
        n, ms, b = C.c_int64(), C.c_double(), C.c_int64()
        L.check(L.lib.cm_comm_profile_read(vg._h, kind, C.byref(n), C.byref(ms), C.byref(b)))
        return int(n.value), float(ms.value)

    # C1
    vg = P.VirtualGroup(4, local, staging_bytes=64 << 20)
    xs = I.c1_inputs()
    ts = [P.Tensor("x", "float32", torch.from_numpy(x).to(device)) for x in xs]
    sha = {c["algo"]: c["sha"] for c in of_kind("c1")}
    res = P.allreduce_group(ts, P.ReduceOp.SUM, vg, algo="auto")
    exact = all(hashlib.sha256(t.to_bytes()).hexdigest() == sha["ring_rsa"] for t, _ in res)
    outs = [torch.empty_like(t.payload) for t in ts]
    st = (L.Stats * 4)()
    ins_a, outs_a = L.ptr_array([t.payload.data_ptr() for t in ts]), L.ptr_array([o.data_ptr() for o in outs])
    stream = torch.cuda.current_stream(device).cuda_stream

    def call():
        L.check(L.lib.cm_allreduce_v(vg._h, ins_a, outs_a, 262144, 0, 0, 0, 131072, 0, stream, st))
    for _ in range(20):
        call()
    torch.cuda.synchronize()
    iters = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        call()
    e1.record()
    torch.cuda.synchronize()
    vg.poll()
    out["c1"] = {"config": "4 ranks x 1 MiB fp32, auto -> ring_rsa, sum", "us_per_call": round(
        e0.elapsed_time(e1) / iters * 1e3, 2), "timing": f"{iters} back-to-back calls, CUDA events, L2-warm",
        "parity": "bit-exact vs reference golden SHA" if exact else "MISMATCH"}
    vg.close()

    # headline kernel configuration at p = 4 and 8
    layers = MODELS["resnet50_like"]
    S = sum(layers) * 4
    for p in (4, 8):
        vg = P.VirtualGroup(p, local, staging_bytes=S + (8 << 20))
        sets = [P.GradientSet(tuple(P.Tensor(nm, "float32", torch.from_numpy(a).to(device))
                                    for nm, a in I.synth_gradients(0, 0, layers, r))) for r in range(p)]
        P.register_gradients_group(sets, vg)
        res = P.aggregate_group(sets, vg)
        parity = None
        for case in of_kind("model"):
            if case["model"] == "resnet50_like" and case["p"] == p:
                h = hashlib.sha256()
                for t in res[0].tensors:
                    h.update(t.to_bytes())
                parity = "bit-exact vs reference golden SHA" if h.hexdigest() == case["sha"] else "MISMATCH"
        if parity is None:
            from oracle import aggregation as OA
            want, _, _ = OA.aggregate([I.synth_gradients(0, 0, layers, r) for r in range(p)], "float32")
            ok = all(t.to_bytes() == want[t.name].tobytes() for t in res[p - 1].tensors)
            parity = "bit-exact vs oracle (reference fold order)" if ok else "MISMATCH"
        for _ in range(3):
            P.aggregate_group(sets, vg)
        torch.cuda.synchronize()
        L.check(L.lib.cm_comm_profile(vg._h, 1))
        k = max(5, min(steps, 20))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            P.aggregate_group(sets, vg)
        e1.record()
        torch.cuda.synchronize()
        n, ms = prof(vg, 0)
        L.check(L.lib.cm_comm_profile(vg._h, 0))
        us = ms / max(n, 1) * 1e3
        alg = 2 * p * S
        ach = alg / (us * 1e-6) / 1e9
        out[f"aggregate_p{p}"] = {
            "config": f"C5 resnet50_like ({S} B fp32 per rank), registered gradients, {p} virtual ranks, "
                      f"one multi-buffer two-shot launch with the fused mean",
            "kernel": "collective_kernel<F32,SUM,MP,ring,MULTI> (SRC_GATHER, bulk-engine reduce)",
            "launches": n, "avg_launch_us": round(us, 2), "step_ms": round(e0.elapsed_time(e1) / k, 4),
            "algorithmic_bytes_per_launch": alg, "achieved": round(ach, 1), "unit": "GB/s",
            "frac": round(ach / pk["hbm_gbs"], 4), "parity": parity,
            "bytes_model": "2*p*S compulsory (gradients read once, means written once); moved incl. staging 3*p*S",
            "moved_bytes_per_launch": 3 * p * S, "traffic": _ncu_traffic(f"virtual_aggregate_p{p}")}
        del sets, res
        vg.close()
        torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------- headline
def headline(args, rank, world, local):
    import paper_1810_11112_b200 as P
    from paper_1810_11112_b200 import _lib as L
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    layers = MODELS[args.model]
    esz = 2 if args.dtype == "bfloat16" else 4
    S = sum(layers) * esz
    comm = P.Communicator(rank, world, local, staging_bytes=max(256 << 20, S + (8 << 20)),
                          pool_bytes=64 << 20, blocking=False)
    for kv in args.param:
        k, v = kv.split("=")
        comm.set_param(k, int(v))
    group = P.GroupSpec(world)
    cfg = P.FusionConfig(args.fusion_threshold)
    gs = make_grads(args.model, rank, device, args.dtype)
    flush_w = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    flush_r = torch.ones(64 << 20, dtype=torch.float32, device=device)

    class _Flush:
        # L2 flush between timed steps (outside the events): write 256 MiB
        # (> 126 MB L2), then read another 256 MiB so the written lines are
        # written back here and L2 holds neither the step's inputs nor dirty
        # lines (the cold, clean state ncu's --cache-control all measures)
        @staticmethod
        def zero_():
            flush_w.zero_()
            flush_r.sum()
    flush = _Flush()

    state = {"out": None, "gs": gs}

    def step():   # persistent output buckets: aggregate(out=previous result)
        state["out"] = P.aggregate(state["gs"], group, comm, algo=args.algo, cfg=cfg,
                                   switch_bytes=args.switch, out=state["out"])
        return state["out"]

    def timed_steps(k):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(k)]
        barrier(world)
        torch.cuda.synchronize()
        for i in range(k):
            flush.zero_()
            ev[i][0].record()
            step()
            ev[i][1].record()
        torch.cuda.synchronize()
        barrier(world)
        return max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in ev), world)

    # unregistered gradients first: plain tensors through the reference API
    # (automatic member registration after the second agreed call, so the
    # warm-up leaves them read in place; packed into staging before that)
    ms_unreg = None
    if world > 1 and not args.no_register:
        for _ in range(args.warmup):
            step()
        ms_unreg = timed_steps(max(10, args.steps // 4))
        # then register the gradient tensors once (collective, outside the
        # timed region): peers read them in place, the pack disappears
        P.register_gradients(gs, comm)
        state["out"] = None

    sampler = ClockSampler(local)
    sampler.start_and_wait()
    for _ in range(args.warmup):
        res = step()
    comm.synchronize()
    parity = oracle_check(args.model, world, rank, res, args.dtype) if (rank == 0 and not args.no_check) else None
    barrier(world)

    nbuf = len(P.fuse_plan(list(gs.tensors), cfg))

    def timed_pass():
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        barrier(world)
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()                   # L2 flush (write 256 MiB > 126 MB L2, then read), untimed
            evs[i][0].record()
            step()
            evs[i][1].record()
        torch.cuda.synchronize()
        barrier(world)
        return statistics.mean(a.elapsed_time(b) for a, b in evs)

    # 1. the headline: EXACTLY K timed steps, nothing else on the stream
    launches0 = comm.launches
    sampler.mark_start()
    ms_local = timed_pass()
    sampler.mark_stop()
    clocks = sampler.result()
    comm.synchronize()
    launches = comm.launches - launches0
    # 2. the roofline: a second pass of K steps with CUDA events around every
    # launch of the library (on its stream), for the per-kernel durations;
    # those bracketing events cost a few us per launch, so the headline above
    # is taken without them
    L.check(L.lib.cm_comm_profile(comm._h, 1))
    ms_prof_local = timed_pass()
    comm.synchronize()

    def prof(kind):
        n, ms, b = C.c_int64(), C.c_double(), C.c_int64()
        L.check(L.lib.cm_comm_profile_read(comm._h, kind, C.byref(n), C.byref(ms), C.byref(b)))
        return int(n.value), float(ms.value), int(b.value)
    coll_n, coll_ms, coll_b = prof(0)
    pack_n, pack_ms, pack_b = prof(1)
    small_n, small_ms, _ = prof(2)          # agreement checks (LL one-shot)
    L.check(L.lib.cm_comm_profile(comm._h, 0))
    ms_prof = max_over_ranks(ms_prof_local, world)
    ms = max_over_ranks(ms_local, world)

    # NCCL comparator on the same fused buffers (N >= 2)
    nccl = None
    if world > 1 and not args.no_nccl:
        sizes = []
        for grp in P.fuse_plan(list(gs.tensors), cfg):
            sizes.append(sum(layers[i] for i in grp))
        bufs = [torch.randn(n, device=device).to(gs.tensors[0].payload.dtype) for n in sizes]
        for _ in range(3):
            for b in bufs:
                dist.all_reduce(b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        reps = max(5, min(args.steps, 50))
        for _ in range(reps):
            flush.zero_()
            e0.record()
            for b in bufs:
                dist.all_reduce(b)
                b.div_(world)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        nccl_ms = max_over_ranks(tot / reps, world)
        nccl = {"ms_per_step": round(nccl_ms, 4), "value": round(world * S / (nccl_ms * 1e-3) / 1e9, 2),
                "what": f"torch.distributed NCCL all_reduce(SUM)+div on the same {len(sizes)} fused buffers"}

    # end-to-end through the public API with pinned host gradients
    e2e = None
    if not args.no_e2e:
        hgs = make_grads(args.model, rank, None, args.dtype, pinned=True)
        comm.blocking = True
        r = None
        for _ in range(2):
            r = P.aggregate(hgs, group, comm, algo=args.algo, cfg=cfg, switch_bytes=args.switch, out=r)
        barrier(world)
        k = max(3, min(args.steps, 20))
        t0 = time.perf_counter()
        for _ in range(k):
            r = P.aggregate(hgs, group, comm, algo=args.algo, cfg=cfg, switch_bytes=args.switch, out=r)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks((time.perf_counter() - t0) / k * 1e3, world)
        assert not r.tensors[0].is_cuda
        e2e = {"value": round(world * S / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": S, "d2h_bytes_per_step": S,
               "what": "aggregate() on pinned host gradients (views of one flat pinned buffer): H2D on a copy stream, fused "
                       "allreduce+mean on the compute stream, D2H on a second copy stream straight "
                       "into pinned host buckets (aggregate(out=prev)), overlapped per fused group; "
                       "host wall clock, max over ranks"}

    pk, pk_src = peaks()
    if world > 1:
        ach = coll_b / (coll_ms * 1e-3) / 1e9 if coll_ms > 0 else 0.0
        ach = max_over_ranks(-ach, world) * -1  # min over ranks (slowest rank)
        roofline = {"bound": "nvlink", "kernel": "collective_kernel (two-shot RS+AG, ring order; one "
                                                   "multi-buffer launch per step)",
                    "achieved": round(ach, 2), "peak": NVLINK_PEAK_GBS, "unit": "GB/s",
                    "frac": round(ach / NVLINK_PEAK_GBS, 4),
                    "peak_source": "B200_PROFILING.md measured NVLink peer copy (900 nominal)",
                    "traffic": None,
                    "algorithmic_bytes_per_launch": coll_b // max(coll_n, 1),
                    "launches": coll_n, "avg_launch_us": round(coll_ms / max(coll_n, 1) * 1e3, 2),
                    "other_launches": {"agreement_check_ll": small_n,
                                       "avg_us": round(small_ms / max(small_n, 1) * 1e3, 2),
                                       "pack": pack_n, "pack_avg_us": round(pack_ms / max(pack_n, 1) * 1e3, 2)},
                    "measured": "second timed pass of K steps with CUDA events around every launch"}
    else:
        ach = pack_b / (pack_ms * 1e-3) / 1e9 if pack_ms > 0 else 0.0
        roofline = {"bound": "hbm", "kernel": "batched_copy_kernel (fused pack, p=1 identity allreduce)",
                    "achieved": round(ach, 2), "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": round(ach / pk["hbm_gbs"], 4), "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_src})",
                    "traffic": _ncu_traffic("batched_copy_kernel"),
                    "algorithmic_bytes_per_launch": pack_b // max(pack_n, 1),
                    "launches": pack_n, "avg_launch_us": round(pack_ms / max(pack_n, 1) * 1e3, 2),
                    "measured": "second timed pass of K steps with CUDA events around every launch"}

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        times = cpu_baseline_sample(args.model, 1, args.dtype)
        t = statistics.median(times)
        cpu = {"value": round(S / t / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "port",
               "sample": f"{len(times)} full steps of the same workload at p=1 (oracle/threaded.py "
                         f"aggregate: np.concatenate fuse, identity allreduce, float64 mean), "
                         f"median {t * 1e3:.1f} ms/step"}

    virt = None
    if world == 1 and rank == 0 and not args.no_virtual:
        virt = virtual_block(args, local, args.steps)

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(world * S / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.dtype == "float32" else "bf16",
            "data": "synthetic: reference synth_gradients recipe (seed 0, iteration 0)",
            "config": {"workload": f"C5 {args.model} gradient set, tensor-fused allreduce + mean per "
                                   f"step (aggregate)",
                       "params_per_rank": sum(layers), "grad_bytes_per_rank": S,
                       "tensors": len(layers), "fused_buffers": nbuf,
                       "fusion_threshold": args.fusion_threshold, "algo": args.algo,
                       "switch_bytes": args.switch, "parallelism": f"dp{world}",
                       "l2": "flushed between timed steps (outside the events): 256 MiB memset, then a 256 MiB read so no dirty lines remain",
                       "outputs": "persistent fused output buckets (aggregate(out=prev))",
                       "gradients": ("registered once with register_gradients (outside the timed "
                                     "region): peers read them in place, no pack")
                       if (world > 1 and not args.no_register) else "unregistered: packed every step"},
            "ms_per_step_unregistered": None if ms_unreg is None else round(ms_unreg, 4),
            "unregistered_what": ("plain tensors through the reference API (no register_gradients): the "
                                  "members are registered automatically after the second agreed aggregate "
                                  "(warm-up), then read in place") if ms_unreg is not None else None,
            "ms_per_step_profiled_pass": round(ms_prof, 4),
            "latency_us": round(ms * 1e3, 2),
            "bus_gbps": round(2 * (world - 1) / world * S / (ms * 1e-3) / 1e9, 2) if world > 1 else None,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "gpu_launches_per_step": launches / max(args.steps, 1),
            "clocks": clocks, "nccl": nccl, "parity": parity,
        }
        if virt is not None:
            out["virtual"] = virt
        emit(out)
    comm.close()


def _ncu_traffic(kernel: str):
    """dram read+write bytes per launch from the committed ncu summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(kernel)
    except (OSError, ValueError):
        return None


# --------------------------------------------------------------- reference arm
def reference_arm(args, rank, world):
    if rank != 0:
        return
    layers = MODELS[args.model]
    S = sum(layers) * 4
    from oracle import threaded as T
    from tests.golden.inputs import synth_gradients
    grads = [synth_gradients(0, 0, layers, r) for r in range(world)]

    def step():
        T.ThreadNet(world).run(lambda r, tp: T.aggregate_rank(grads[r], tp, algo=args.algo))

    for _ in range(min(args.warmup, 1)):
        step()
    budget = args.ref_budget_s
    times = []
    t_start = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget:
            break
    ms = statistics.mean(times) * 1e3
    val = round(world * S / (ms * 1e-3) / 1e9, 4)
    cores = min(world, os.cpu_count() or 1)
    out = {
        "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": world, "steps": len(times),
        "steps_requested": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: reference synth_gradients recipe (seed 0, iteration 0)",
        "config": {"workload": f"C5 {args.model} gradient set, tensor-fused allreduce + mean per step "
                               f"(aggregate)", "params_per_rank": sum(layers), "grad_bytes_per_rank": S,
                   "fusion_threshold": 67108864, "algo": args.algo, "parallelism": f"dp{world}"},
        "impl": "reference",
        "cpu_baseline": {"value": val, "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"{len(times)} full steps; {world} rank threads of oracle/threaded.py "
                                   f"(message-passing restatement of collectives.py ring/rhd + "
                                   f"aggregation.py, numpy) on host cores"},
        "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(out)


# ------------------------------------------------------------------ sweep/tune
def _time_calls(fn, iters, warmup, graph=False):
    """Device ms per call: CUDA events around `iters` back-to-back calls, or a
    CUDA graph of `iters` calls replayed once."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(iters):
                    fn()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
    else:
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def sweep(args, rank, world, local):
    import paper_1810_11112_b200 as P
    from paper_1810_11112_b200 import _lib as L
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    maxb = args.sweep_max
    comm = P.Communicator(rank, world, local, staging_bytes=max(64 << 20, maxb + (4 << 20)),
                          pool_bytes=max(64 << 20, 2 * maxb + (4 << 20)), blocking=False)
    st = L.Stats()
    rows = []
    sizes = []
    b = args.sweep_min
    while b <= maxb:
        sizes.append(b)
        b *= 2
    for kv in args.param:
        k, v = kv.split("=")
        comm.set_param(k, int(v))
    src = comm.empty(maxb // 4, "float32")
    dst = comm.empty(maxb // 4, "float32")
    plain = torch.randn(maxb // 4, device=device)
    plain_out = torch.empty_like(plain)
    src.normal_()
    stream = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731

    def ours(n, algo, zc):
        s, d = (src, dst) if zc else (plain, plain_out)
        return lambda: L.check(L.lib.cm_allreduce(comm._h, s.data_ptr(), d.data_ptr(), n,
                                                  0, 0, L.ALGO[algo], args.switch or 131072, 0,
                                                  stream(), C.byref(st)))
    for nbytes in sizes:
        n = max(1, nbytes // 4)
        iters = 200 if nbytes <= (1 << 20) else (50 if nbytes <= (64 << 20) else 10)
        row = {"message_bytes": nbytes, "p": world}
        for algo in args.algos.split(","):
            barrier(world)
            row[f"{algo}_us"] = max_over_ranks(_time_calls(ours(n, algo, False), iters, 5) * 1e3, world)
            barrier(world)
            row[f"{algo}_zc_us"] = max_over_ranks(_time_calls(ours(n, algo, True), iters, 5) * 1e3, world)
            if nbytes <= (4 << 20):
                barrier(world)
                row[f"{algo}_graph_us"] = max_over_ranks(
                    _time_calls(ours(n, algo, True), iters, 3, graph=True) * 1e3, world)
        comm.synchronize()
        if world > 1 and not args.no_nccl:
            t = plain[:n]
            barrier(world)
            row["nccl_us"] = max_over_ranks(_time_calls(lambda: dist.all_reduce(t), iters, 5) * 1e3, world)
            if nbytes <= (4 << 20):
                barrier(world)
                row["nccl_graph_us"] = max_over_ranks(
                    _time_calls(lambda: dist.all_reduce(t), iters, 3, graph=True) * 1e3, world)
        best = min(row[f"{a}{v}_us"] for a in args.algos.split(",") for v in ("", "_zc"))
        row["best_us"] = best
        fac = 2 * (world - 1) / world if world > 1 else 0.0
        row["bus_gbps"] = round(nbytes * fac / (best * 1e-6) / 1e9, 3)
        row["roofline_frac"] = round(row["bus_gbps"] / NVLINK_PEAK_GBS, 4)
        if "nccl_us" in row:
            row["nccl_bus_gbps"] = round(nbytes * fac / (row["nccl_us"] * 1e-6) / 1e9, 3)
        rows.append(row)
        if rank == 0:
            log(json.dumps(row))
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        path = args.out or os.path.join(ROOT, "gpurun_out", f"sweep_p{world}.csv")
        keys = sorted({k for r in rows for k in r}, key=lambda k: (k != "message_bytes", k != "p", k))
        with open(path, "w") as fh:
            fh.write(",".join(keys) + "\n")
            for r in rows:
                fh.write(",".join(format(r.get(k, ""), ".6g") if isinstance(r.get(k), float)
                                  else str(r.get(k, "")) for k in keys) + "\n")
        emit({"mode": "sweep", "p": world, "rows": rows})
    comm.close()


def tune(args, rank, world, local):
    """Measure, per message size, rhd one-shot (LL), rhd two-shot, ring (LL
    two-shot while the segments fit the LL slots) and ring on the pull kernel,
    all CUDA-graph timed, and store per group size: the largest size worth
    reducing one-shot (oneshot_max_bytes = ll_max_bytes), the largest size
    worth the LL two-shot (ll2_max_bytes) and the switch point from which
    ring_rsa beats rhd_rsa (collectives.py:239-247's threshold, measured on
    this box) in paper_1810_11112_b200/tuning.json."""
    import paper_1810_11112_b200 as P
    from paper_1810_11112_b200 import _lib as L
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    comm = P.Communicator(rank, world, local, staging_bytes=64 << 20, pool_bytes=64 << 20, blocking=False)
    x = torch.randn(8 << 20, device=device)
    y = torch.empty_like(x)
    st = L.Stats()
    sizes = [1 << k for k in range(10, 24)]
    res = {}
    big = 1 << 40
    for nbytes in sizes:
        n = nbytes // 4
        t = {}
        for name, algo, osm, ll2 in (("rhd_oneshot", "rhd_rsa", big, big), ("rhd_twoshot", "rhd_rsa", 1, big),
                                     ("ring", "ring_rsa", big, big), ("ring_pull", "ring_rsa", big, 1)):
            comm.set_param("oneshot_max_bytes", osm)
            comm.set_param("ll_max_bytes", osm)
            comm.set_param("ll2_max_bytes", ll2)
            fn = lambda a=algo: L.check(L.lib.cm_allreduce(  # noqa: E731
                comm._h, x.data_ptr(), y.data_ptr(), n, 0, 0, L.ALGO[a], 131072, 0,
                torch.cuda.current_stream().cuda_stream, C.byref(st)))
            barrier(world)
            t[name] = max_over_ranks(_time_calls(fn, 100, 5, graph=True) * 1e3, world)
        res[nbytes] = t
        if rank == 0:
            log(json.dumps({"bytes": nbytes, **{k: round(v, 2) for k, v in t.items()}}))
    oneshot_max = 0
    for nbytes in sizes:
        if res[nbytes]["rhd_oneshot"] <= res[nbytes]["rhd_twoshot"]:
            oneshot_max = nbytes
        else:
            break
    ll2_max = 0
    for nbytes in sizes:
        if res[nbytes]["ring"] <= res[nbytes]["ring_pull"]:
            ll2_max = nbytes
        else:
            break

    def rhd_best(b):
        return res[b]["rhd_oneshot"] if b <= oneshot_max else res[b]["rhd_twoshot"]
    switch = None
    for nbytes in sizes:
        if res[nbytes]["ring"] < rhd_best(nbytes):
            switch = nbytes
            break
    if switch is None:
        switch = 1 << 24
    if rank == 0:
        path = os.path.join(ROOT, "paper_1810_11112_b200", "tuning.json")
        try:
            with open(path) as fh:
                data = json.load(fh)
        except (OSError, ValueError):
            data = {}
        data.setdefault("switch_bytes", {})[str(world)] = switch
        data.setdefault("oneshot_max_bytes", {})[str(world)] = max(oneshot_max, 1024)
        data.setdefault("ll2_max_bytes", {})[str(world)] = max(ll2_max, 1024)
        data.setdefault("measured_us_cuda_graph", {})[str(world)] = {
            str(k): {a: round(v, 3) for a, v in t.items()} for k, t in res.items()}
        data["how"] = "bench.py --mode tune on a B200 box: CUDA-graph timed, max over ranks"
        with open(path, "w") as fh:
            json.dump(data, fh, indent=1)
        emit({"mode": "tune", "p": world, "switch_bytes": switch, "oneshot_max_bytes": oneshot_max,
              "ll2_max_bytes": ll2_max})
    comm.close()


def refsweep(args):
    """Reference CPU path per message size: oracle/threaded.py (the
    reference's message-passing ring/rhd programs, numpy, one thread per
    rank) for p = --ranks, float32, timed on this host. CSV to stdout."""
    from oracle import threaded as T
    p = args.ranks
    rows = ["message_bytes,p,algo,mean_ms,min_ms,iters"]
    b = args.sweep_min
    while b <= args.sweep_max:
        n = max(1, b // 4)
        rng = np.random.default_rng([0, b])
        xs = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
        algo = "rhd_rsa" if b < 131072 else "ring_rsa"
        times = []
        t_end = time.perf_counter() + 3.0
        while len(times) < 50 and (time.perf_counter() < t_end or len(times) < 2):
            t0 = time.perf_counter()
            T.ThreadNet(p).run(lambda r, tp: T.allreduce_rank(xs[r], "sum", algo, tp))
            times.append(time.perf_counter() - t0)
        rows.append(f"{b},{p},{algo},{statistics.mean(times) * 1e3:.4f},{min(times) * 1e3:.4f},{len(times)}")
        log(rows[-1])
        b *= 4
    emit({"mode": "refsweep", "p": p, "csv": rows})


def overlap(args, rank, world, local):
    """Caller-side study: a synthetic backward pass (one
    bf16 GEMM per layer on the producer stream, last layer first) producing the
    C5 gradients, aggregated (A) after the backward pass with aggregate() or
    (B) overlapped with it through OverlappedAggregator. Step = backward +
    aggregation, CUDA events, max over ranks; results checked equal."""
    import paper_1810_11112_b200 as P
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    layers = MODELS[args.model]
    S = sum(layers) * 4
    comm = P.Communicator(rank, world, local, staging_bytes=max(256 << 20, S + (8 << 20)),
                          pool_bytes=64 << 20, blocking=False)
    for kv in args.param:
        k, v = kv.split("=")
        comm.set_param(k, int(v))
    group = P.GroupSpec(world)
    cfg = P.FusionConfig(args.fusion_threshold)
    src = make_grads(args.model, rank, device)
    names = [t.name for t in src.tensors]
    grads = [torch.empty_like(t.payload) for t in src.tensors]
    gdim = args.gemm
    wts = [torch.randn(gdim, gdim, device=device, dtype=torch.bfloat16) for _ in range(2)]

    def layer_compute():
        torch.matmul(wts[0], wts[1])

    def backward(ov=None):
        for i in reversed(range(len(grads))):
            layer_compute()
            grads[i].copy_(src.tensors[i].payload)
            if ov is not None:
                ov.ready(names[i], grads[i])

    gs_view = P.GradientSet(tuple(P.Tensor(nm, "float32", g) for nm, g in zip(names, grads)))
    ov = P.OverlappedAggregator(gs_view, comm, algo=args.algo, cfg=cfg, max_ctas=args.ov_ctas or None,
                                priority=args.ov_priority, cluster_pairs=bool(args.ov_pairs),
                                pack_ctas=args.ov_pack_ctas or None, register_members=bool(args.ov_register))

    def step_seq():
        backward()
        return P.aggregate(gs_view, group, comm, algo=args.algo, cfg=cfg)

    def step_ovl():
        backward(ov)
        return ov.finish()

    def step_bwd():
        backward()

    def timed(fn, k):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            r = fn()
        e1.record()
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1) / k, world), r

    k = max(5, min(args.steps, 30))
    t_bwd, _ = timed(step_bwd, k)
    t_seq, r_seq = timed(step_seq, k)
    if args.gemm_carveout:      # the overlapped backward leaves SMs to the collectives
        torch._C._set_sm_carveout_experimental(args.gemm_carveout)
    try:
        t_ovl, r_ovl = timed(step_ovl, k)
        t_bwd_cv = timed(step_bwd, k)[0] if args.gemm_carveout else t_bwd
    finally:
        if args.gemm_carveout:
            torch._C._set_sm_carveout_experimental(None)
    if os.environ.get("CM_OVERLAP_TRACE") and rank == 0:
        # one overlapped step under torch.profiler (CUPTI kernel timeline), diagnostics only
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step_ovl()
            torch.cuda.synchronize()
        prof.export_chrome_trace(os.environ["CM_OVERLAP_TRACE"])
    elif os.environ.get("CM_OVERLAP_TRACE"):
        step_ovl()
        torch.cuda.synchronize()
    same = all(a.to_bytes() == b.to_bytes() for a, b in zip(r_seq.tensors, r_ovl.tensors))
    comm.synchronize()
    if rank == 0:
        emit({"mode": "overlap", "n_gpus": world, "model": args.model, "gemm": gdim,
              "backward_ms": round(t_bwd, 4), "sequential_ms": round(t_seq, 4), "overlapped_ms": round(t_ovl, 4),
              "hidden_frac": round((t_seq - t_ovl) / max(t_seq - t_bwd, 1e-9), 3),
              "groups": len(ov.groups), "ov_ctas": args.ov_ctas, "ov_priority": args.ov_priority,
              "gemm_carveout": args.gemm_carveout, "backward_carveout_ms": round(t_bwd_cv, 4),
              "ov_pairs": args.ov_pairs, "ov_pack_ctas": args.ov_pack_ctas, "ov_register": args.ov_register,
              "bit_identical": same})
    comm.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--mode", choices=("headline", "sweep", "tune", "refsweep", "overlap"), default="headline")
    ap.add_argument("--gemm", type=int, default=2048, help="overlap: per-layer bf16 GEMM size")
    ap.add_argument("--ov-ctas", type=int, default=64, help="overlap: CTA cap of overlapped collectives (0: none)")
    ap.add_argument("--ov-priority", type=int, default=0, help="overlap: communication stream priority (-1: high)")
    ap.add_argument("--ov-pairs", type=int, default=0, help="overlap: capped grids in 2-CTA clusters (1: on)")
    ap.add_argument("--ov-pack-ctas", type=int, default=0, help="overlap: CTA cap of the member pack (0: none)")
    ap.add_argument("--ov-register", type=int, default=0,
                    help="overlap: register the persistent gradient buffers after the first step (1: on)")
    ap.add_argument("--gemm-carveout", type=int, default=0,
                    help="overlap: SMs the backward GEMMs leave free while the collectives overlap them "
                         "(cuBLAS SM carve-out, overlapped step only; 0: none)")
    ap.add_argument("--ranks", type=int, default=4, help="refsweep: simulated ranks")
    ap.add_argument("--model", choices=tuple(MODELS), default="resnet50_like")
    ap.add_argument("--dtype", choices=("float32", "bfloat16"), default="float32")
    ap.add_argument("--algo", default="auto")
    ap.add_argument("--switch", type=int, default=None, help="switch_bytes (default: measured table)")
    ap.add_argument("--fusion-threshold", type=int, default=67108864)
    ap.add_argument("--sweep-min", type=int, default=4)
    ap.add_argument("--sweep-max", type=int, default=1 << 30)
    ap.add_argument("--ref-budget-s", type=float, default=90.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-virtual", action="store_true", help="N=1: skip the virtual-group kernel block")
    ap.add_argument("--no-register", action="store_true",
                    help="do not register the gradient tensors (pack them every step)")
    ap.add_argument("--param", action="append", default=[],
                    help="communicator tuning knob key=value (cm_comm_set_param)")
    ap.add_argument("--algos", default="rhd_rsa,ring_rsa", help="sweep: algorithms to time")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    _isolate_stdout()
    rank, world, local = dist_env()
    if args.gpus is not None and args.gpus != world:
        log(f"note: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE")
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if args.mode == "refsweep":
        if rank == 0:
            refsweep(args)
        return
    init_dist(rank, world, local, nccl=True)
    try:
        if args.mode == "headline":
            headline(args, rank, world, local)
        elif args.mode == "sweep":
            sweep(args, rank, world, local)
        elif args.mode == "overlap":
            overlap(args, rank, world, local)
        else:
            tune(args, rank, world, local)
    finally:
        if world > 1 and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
