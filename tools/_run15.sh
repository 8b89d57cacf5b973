timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q 2>&1 | tail -2
for n in 2 4; do for b in 101760000 1073741824; do timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29621 tools/phase_trace.py --bytes $b --zc 2>/dev/null | grep "p="; done; done
for n in 2 4; do timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $n --no-e2e > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo rc=$?; done
for n in 2 4; do python - <<PY
import json
d=json.loads(open("gpurun_out/bench_n$n.json").read().strip().splitlines()[-1]); r=d["roofline"]
print($n, d["value"], d["ms_per_step"], d.get("ms_per_step_unregistered"), r["achieved"], r["frac"], r["avg_launch_us"], (d.get("nccl") or {}).get("ms_per_step"))
PY
done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -2
