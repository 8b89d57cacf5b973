#!/bin/bash
# Round-2 closing pass on a 4-GPU box: every GPU test tier, then the bench
# lines at N = 1, 2, 4 and the reference arm at N = 1.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final2_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/final2_tests.log
timeout 900 python bench.py > gpurun_out/final2_n1.json 2> gpurun_out/final2_n1.err; echo "n1 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2964$n bench.py --gpus $n > gpurun_out/final2_n$n.json 2> gpurun_out/final2_n$n.err; echo "n$n rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/final2_ref_n1.json 2> gpurun_out/final2_ref_n1.err; echo "ref rc=$?"
