#!/bin/bash
# same-box A/B of the headline step under knob settings: ab_headline.sh N "k=v,k=v" "k=v" ...
# ("-" = defaults); two rounds, 50 steps each
N=$1; shift
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29960
for rep in 1 2; do
  for cfg in "$@"; do
    port=$((port+1))
    args=""
    [ "$cfg" != "-" ] && args=$(echo $cfg | tr ',' '\n' | sed 's/^/--param /' | tr '\n' ' ')
    $T --master-port $port bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --no-nccl $args > gpurun_out/ab.json 2>/dev/null
    python - "$cfg" "$rep" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:<34} rep={sys.argv[2]} ms/step={d['ms_per_step']} unreg={d['ms_per_step_unregistered']} "
      f"kernel_us={d['roofline']['avg_launch_us']} busbw={d['bus_gbps']}")
PY
  done
done
