for n in 2 4; do timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29621 tools/phase_trace.py --agg 2>&1 | grep "p=" | cut -c1-300; done
