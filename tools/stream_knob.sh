#!/bin/bash
# pipelined two-shot (stream_chunk: per-warp reduce progress, allgather warps
# pull chunk k while chunk k+1 is reduced) vs the barrier two-shot, p = N GPUs
N=${1:-4}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29770
for cfg in "" "stream_chunk=4096" "stream_chunk=16384" "stream_chunk=65536"; do
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
