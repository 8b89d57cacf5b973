timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q -k "rhd_logp" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -5
for n in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n --mode sweep --sweep-min 4 --sweep-max 16777216 --algos rhd_rsa --param rhd_logp=2 --out gpurun_out/sweep_logp_p$n.csv > /dev/null 2>gpurun_out/sweep_logp_p$n.err; echo rc=$?
done
