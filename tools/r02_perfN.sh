#!/bin/bash
# round-2 N-GPU perf pass (gpurun --gpus N): headline, C2/C3 sweep (plain vs symmetric buffers,
# NCCL via torch), pointer-cache A/B, direct NCCL comparator (NVLS default / off)
N=${1:-4}
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
$T --master-port 29711 bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/r02_bench_n$N.json 2> gpurun_out/r02_bench_n$N.err; echo "bench rc=$?"
$T --master-port 29712 bench.py --gpus $N --mode sweep --out gpurun_out/r02_sweep_p$N.csv > /dev/null 2> gpurun_out/r02_sweep_p$N.err; echo "sweep rc=$?"
$T --master-port 29713 tools/ptrcache_ab.py --out gpurun_out/r02_ptrcache_ab_p$N.txt > /dev/null 2> gpurun_out/r02_ptrcache_p$N.err; echo "ptrcache rc=$?"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING $T --master-port 29714 tools/nccl_direct.py --out gpurun_out/r02_nccl_direct_p$N.csv > gpurun_out/r02_nccl_direct_p$N.log 2>&1; echo "nccl rc=$?"
NCCL_NVLS_ENABLE=0 NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING $T --master-port 29715 tools/nccl_direct.py --out gpurun_out/r02_nccl_direct_nonvls_p$N.csv > gpurun_out/r02_nccl_direct_nonvls_p$N.log 2>&1; echo "nccl nonvls rc=$?"
