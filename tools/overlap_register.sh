#!/bin/bash
# Overlapped aggregation (N=4): member pack every step vs members registered
# after the first step (peers read the persistent gradient buffers in place)
port=29880
for rep in 1 2; do
for cfg in "0 2048" "1 2048" "0 4096" "1 4096"; do
  set -- $cfg
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --mode overlap --fusion-threshold 16777216 --ov-register $1 --gemm $2 --steps 30 2>/dev/null | grep overlap | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ov_register', d['ov_register'], 'gemm', d['gemm'], 'backward', d['backward_ms'], 'sequential', d['sequential_ms'], 'overlapped', d['overlapped_ms'], 'hidden', d['hidden_frac'], 'bit_identical', d['bit_identical'])"
done
done
