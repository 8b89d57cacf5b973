#!/bin/bash
# medium-message knob study (p = N GPUs): 2..64 MiB, ring_rsa, eager, CUDA events
N=${1:-4}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29750
for cfg in "" "max_ctas=64" "max_ctas=96" "bulk_stage_kb=32" "bulk_stage_kb=16" "twoshot_bytes_per_cta=16384" "ll2_max_bytes=2097152"; do
  port=$((port+1))
  args=$(echo $cfg | tr ',' '\n' | grep . | sed 's/^/--param /' | tr '\n' ' ')
  $T --master-port $port bench.py --gpus $N --mode sweep --sweep-min 2097152 --sweep-max 67108864 --algos ring_rsa \
     --no-nccl $args --out gpurun_out/knob.csv > /dev/null 2>&1
  python - "$cfg" <<'PY'
import csv, sys
rows = list(csv.DictReader(open("gpurun_out/knob.csv")))
print(f"{sys.argv[1] or 'default':<28}", " ".join(f"{int(r['message_bytes'])>>20}M:{float(r['ring_rsa_zc_us']):.1f}" for r in rows))
PY
done
