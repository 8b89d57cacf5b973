for b in 262144 1048576 4194304 16777216; do
 for prm in "max_ctas=148" "ll2_max_bytes=1"; do
  timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 tools/phase_trace.py --bytes $b --zc --param $prm 2>/dev/null | grep "p="
 done
done
