#!/bin/bash
# Overlapped aggregation (N=4): communication stream priority (-1 high, 0 normal) and CTA cap, GEMM 2048^3 / 4096^3
port=29890
for rep in 1 2; do
for cfg in "-1 64 2048" "0 64 2048" "-1 64 4096" "0 64 4096" "0 32 4096"; do
  set -- $cfg
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --mode overlap --fusion-threshold 16777216 --ov-priority=$1 --ov-ctas $2 --gemm $3 --steps 30 2>/dev/null | grep overlap | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prio', d['ov_priority'], 'ctas', d['ov_ctas'], 'gemm', d['gemm'], 'backward', d['backward_ms'], 'sequential', d['sequential_ms'], 'overlapped', d['overlapped_ms'], 'hidden', d['hidden_frac'], 'bit_identical', d['bit_identical'])"
done
done
