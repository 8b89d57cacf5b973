#!/bin/bash
# round-2 2-GPU perf pass (gpurun --gpus 2): headline N=2, C2/C3 sweep (plain vs symmetric
# buffers, NCCL via torch), pointer-cache A/B, direct NCCL comparator (NVLS default / off)
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29701 bench.py --gpus 2 --steps 30 --warmup 5 > gpurun_out/r02_bench_n2.json 2> gpurun_out/r02_bench_n2.err; echo "bench rc=$?"
$T --master-port 29702 bench.py --gpus 2 --mode sweep --out gpurun_out/r02_sweep_p2.csv > /dev/null 2> gpurun_out/r02_sweep_p2.err; echo "sweep rc=$?"
$T --master-port 29703 tools/ptrcache_ab.py --out gpurun_out/r02_ptrcache_ab_p2.txt > /dev/null 2> gpurun_out/r02_ptrcache_p2.err; echo "ptrcache rc=$?"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING $T --master-port 29704 tools/nccl_direct.py --out gpurun_out/r02_nccl_direct_p2.csv > gpurun_out/r02_nccl_direct_p2.log 2>&1; echo "nccl rc=$?"
NCCL_NVLS_ENABLE=0 NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING $T --master-port 29705 tools/nccl_direct.py --out gpurun_out/r02_nccl_direct_nonvls_p2.csv > gpurun_out/r02_nccl_direct_nonvls_p2.log 2>&1; echo "nccl nonvls rc=$?"
