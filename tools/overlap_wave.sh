#!/bin/bash
# Overlapped aggregation (N=4): CTA cap that leaves exactly one GEMM wave (148 - 128 = 20 SMs, whole TPCs) vs 64
port=29900
for rep in 1 2; do
for cfg in "64 0 4096" "20 1 4096" "64 0 2048" "20 1 2048"; do
  set -- $cfg
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --mode overlap --fusion-threshold 16777216 --ov-ctas $1 --ov-pairs $2 --gemm $3 --steps 30 2>/dev/null | grep overlap | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ctas', d['ov_ctas'], 'pairs', d['ov_pairs'], 'gemm', d['gemm'], 'backward', d['backward_ms'], 'sequential', d['sequential_ms'], 'overlapped', d['overlapped_ms'], 'hidden', d['hidden_frac'], 'bit_identical', d['bit_identical'])"
done
done
