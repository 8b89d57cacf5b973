python tools/pcie_bw.py 2>&1 | grep rank
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 tools/pcie_bw.py 2>&1 | grep rank
