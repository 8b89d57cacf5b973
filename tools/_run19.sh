timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_virtual.py -x -q 2>&1 | tail -2
REG=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 tools/timeline.py 2>&1 | grep -v "^W1\|Warn\|warn\|\*\*\*\|OMP" | head -12
for n in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $n --no-e2e > gpurun_out/bench_n$n.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_n$n.json').read().strip().splitlines()[-1]); r=d['roofline']; print('n=$n', d['ms_per_step'], d.get('ms_per_step_unregistered'), r['frac'], r['avg_launch_us'], d['nccl']['ms_per_step'], d['parity'])"; done
