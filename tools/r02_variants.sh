#!/bin/bash
# headline variants on N GPUs: bf16 ResNet-50 set, MobileNet set (config 4), fp32 ResNet-50 (config 5)
N=${1:-4}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29930
for v in "--model resnet50_like" "--model resnet50_like --dtype bfloat16" "--model mobilenet_like"; do
  port=$((port+1))
  $T --master-port $port bench.py --gpus $N --steps 30 --warmup 5 --no-e2e $v > gpurun_out/var.json 2>/dev/null
  python - "$v" "$N" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/var.json").read().strip().splitlines()[-1])
nc = d.get("nccl") or {}
print(f"N={sys.argv[2]} {sys.argv[1]:<40} step {d['ms_per_step']} ms (unregistered {d['ms_per_step_unregistered']}), "
      f"busBW {d['bus_gbps']} GB/s, NCCL all_reduce+div {nc.get('ms_per_step')} ms, {d['parity']}")
PY
done
