timeout 300 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo rc=$?
for n in 2 4; do timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo rc=$?; done
for n in 1 2 4; do python - <<PY
import json
d=json.loads(open("gpurun_out/bench_n$n.json").read().strip().splitlines()[-1]); r=d["roofline"]
print($n, d["value"], d["ms_per_step"], d.get("ms_per_step_unregistered"), r["achieved"], r["frac"], r["avg_launch_us"], (d.get("nccl") or {}).get("ms_per_step"), (d.get("e2e") or {}).get("ms_per_step"), (d.get("cpu_baseline") or {}).get("value"), d["clocks"])
PY
done
