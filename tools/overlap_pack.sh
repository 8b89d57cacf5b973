# Overlapped aggregation (N=4): CTA cap of the member pack next to the backward
# GEMMs (the pack otherwise floods every SM for ~8 us per group)
for cfg in "64 0" "64 64" "32 32" "20 20" "32 16"; do
  set -- $cfg
  timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29871 bench.py --gpus 4 --mode overlap --fusion-threshold 16777216 --ov-ctas $1 --ov-pack-ctas $2 --steps 30 2>/dev/null | grep overlap | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ov_ctas', d['ov_ctas'], 'pack_ctas', d['ov_pack_ctas'], 'backward', d['backward_ms'], 'sequential', d['sequential_ms'], 'overlapped', d['overlapped_ms'], 'hidden', d['hidden_frac'], 'bit_identical', d['bit_identical'])"
done
