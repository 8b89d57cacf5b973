#!/bin/bash
# Recipes behind the numbers in profiles/ and BASELINE.md section 5 (run through
# gpurun on a B200 box from the repo root; one gpurun call at a time).
set -x
case "$1" in
  tests)      # parity tiers: 1-GPU virtual groups, then 2/4-GPU processes
    python -m pytest tests -m gpu -x -q ;;
  headline)   # BENCH line at N=1, 2, 4 (one process per GPU)
    python bench.py > gpurun_out/bench_n1.json
    for n in 2 4; do
      python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 2954$n bench.py --gpus $n > gpurun_out/bench_n$n.json
    done ;;
  sweep)      # C2/C3 latency and busBW vs NCCL (profiles/r01_sweep_p{2,4}.csv)
    for n in 2 4; do
      python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 2955$n bench.py --gpus $n --mode sweep --out gpurun_out/sweep_p$n.csv
    done ;;
  ncu)        # launch list + full capture of the N=1 pack and a virtual p=4 collective
    B="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-check"
    $B > /dev/null &&
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/r01_launches_bench_n1.csv $B > /dev/null &&
    ncu --set full --clock-control none --import-source on -k regex:batched_copy -s 6 -c 1 -o /tmp/pack $B &&
    ncu -i /tmp/pack.ncu-rep --page raw --csv > gpurun_out/ncu_pack_raw.csv
    V="python tools/virtual_ar.py --p 4 --n 16320000 --algo ring_rsa --iters 3"
    $V && ncu --set full --clock-control none --import-source on -k regex:collective_kernel -s 1 -c 1 \
        -o /tmp/coll $V && ncu -i /tmp/coll.ncu-rep --page raw --csv > gpurun_out/ncu_coll_raw.csv ;;
  phases)     # per-phase device timing of the headline collective (tools/phase_trace.py)
    for n in 2 4; do
      python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 2962$n tools/phase_trace.py --agg
    done ;;
  overlap)    # overlapped aggregation study (profiles/r01_overlap_n4.txt)
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 29591 bench.py --gpus 4 --mode overlap --fusion-threshold 16777216 ;;
  ps)         # parameter-server step: virtual p=2/4/8, real p=2, kernel launch list (profiles/r01_ps_ab.txt)
    for p in 2 4 8; do python tools/ps_bench.py --p $p; done
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29533 tools/ps_bench.py
    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ps_kernel --csv \
      --log-file gpurun_out/ps_launches.csv python tools/ps_bench.py --p 4 --iters 3 > /dev/null ;;
  hostov)     # small-allreduce host submission vs device drain (profiles/r01_host_overhead_p2.txt)
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29561 tools/host_overhead.py ;;
  pcie)       # host copy ceilings behind the e2e number
    python tools/pcie_bw.py
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 29571 tools/pcie_bw.py ;;
  *) echo "usage: $0 tests|headline|sweep|ncu|phases|overlap|pcie"; exit 2 ;;
esac
