timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; tail -2 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo rc=$?
for n in 2 4; do timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo rc=$?; done
timeout 400 python bench.py --impl reference > gpurun_out/ref_n1.json 2>/dev/null; echo rc=$?
for n in 2 4; do timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n bench.py --impl reference --gpus $n > gpurun_out/ref_n$n.json 2>/dev/null; echo rc=$?; done
for n in 1 2 4; do python - <<PY
import json
d=json.loads(open("gpurun_out/bench_n$n.json").read().strip().splitlines()[-1]); r=d["roofline"]
ref=json.loads(open("gpurun_out/ref_n$n.json").read().strip().splitlines()[-1])
print($n, d["value"], d["ms_per_step"], d.get("ms_per_step_unregistered"), r["frac"], (d.get("nccl") or {}).get("ms_per_step"), d["e2e"]["ms_per_step"], d["e2e"]["value"], (d.get("cpu_baseline") or {}).get("value"), d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], "ref", ref.get("value"), ref.get("ms_per_step"))
PY
done
