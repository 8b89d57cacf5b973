timeout 600 python -m pytest tests/test_gpu_virtual.py -x -q 2>&1 | tail -2
for n in 2 4; do for d in 2 1 2 1; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $n --no-e2e --no-nccl --no-check --param dyn_ag=$d > gpurun_out/bx.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bx.json').read().strip().splitlines()[-1]); r=d['roofline']; print('n=$n dyn=$d', d['ms_per_step'], d.get('ms_per_step_unregistered'), r['frac'], r['avg_launch_us'])"; done; done
for n in 2 4; do timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29621 tools/phase_trace.py --agg 2>&1 | grep "p=" | cut -c1-300; done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -2
