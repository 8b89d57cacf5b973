# Overlapped aggregation (bench.py --mode overlap) at N=4: CTA cap of the
# overlapped collectives, with and without 2-CTA clusters (whole TPCs next to
# the 2-SM-cluster GEMMs of the synthetic backward); the last group runs uncapped.
for cfg in "64 0" "64 1" "32 1" "24 1" "20 1" "16 1" "20 0"; do
  set -- $cfg
  timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29871 bench.py --gpus 4 --mode overlap --fusion-threshold 16777216 --ov-ctas $1 --ov-pairs $2 --steps 30 2>/dev/null | grep overlap
done
