#!/bin/bash
# same-box A/B of the overlapped two-shot (multi-buffer headline), N = number of GPUs;
# extra args: overlap_chunks values to try
N=${1:-2}; shift
CH=${@:-4}
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29700
for rep in 1 2; do
  for cfg in "overlap=1" $(for c in $CH; do echo "overlap=2,overlap_chunks=$c"; done); do
    port=$((port+1))
    args=$(echo $cfg | tr ',' '\n' | sed 's/^/--param /' | tr '\n' ' ')
    $T --master-port $port bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --no-nccl $args \
      > gpurun_out/ab_ovl.json 2>/dev/null
    python - "$cfg" "$rep" gpurun_out/ab_ovl.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
print(f"{sys.argv[1]:<32} rep={sys.argv[2]} ms/step={d['ms_per_step']} unreg={d['ms_per_step_unregistered']} "
      f"kernel_us={d['roofline']['avg_launch_us']} busbw={d['bus_gbps']}")
PY
  done
done
