timeout 600 python -m pytest tests/test_gpu_virtual.py -x -q -k "overlapped or single_rank" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "two or four" 2>&1 | tail -2
for n in 2 4; do for prm in "max_ctas=148" "max_ctas=64" "max_ctas=32"; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus $n --mode overlap --fusion-threshold 16777216 --param $prm 2>/dev/null | sed "s/^/$prm /"; done; done
