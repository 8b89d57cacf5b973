#!/bin/bash
# Host-gradient pipeline at N GPUs: fused groups in host_chunk pieces (host_split=2)
# vs one launch per group (host_split=1); e2e ms per step, same box, alternating
N=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29810
for rep in 1 2; do
  for cfg in "host_split=1" "host_piece_kb=1024" "host_piece_kb=2048" "host_piece_kb=4096"; do
    port=$((port+1))
    args=$(echo $cfg | tr ',' '\n' | sed 's/^/--param /' | tr '\n' ' ')
    timeout 300 $T --master-port $port bench.py --gpus $N --steps 20 --warmup 3 --no-cpu $args 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N $cfg', 'e2e_ms', d['e2e']['ms_per_step'], 'step_ms', d['ms_per_step'])"
  done
done
