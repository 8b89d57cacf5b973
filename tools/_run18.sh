REG=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 tools/timeline.py 2>&1 | grep -v "^W1\|Warn\|warn" | head -30
