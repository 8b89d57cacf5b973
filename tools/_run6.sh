python tools/pcie_bw.py 2>&1 | grep rank
for n in 2 4; do timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29551 tools/pcie_bw.py 2>&1 | grep rank; done
nvidia-smi topo -m 2>&1 | head -20
numactl -H 2>&1 | head -5; lscpu | grep -i "numa\|model name\|socket"
