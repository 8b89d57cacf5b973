mkdir -p gpurun_out/t2
i=0
for n in 4 2; do
for prm in "max_ctas=148" "ll2_max_bytes=1" "ll2_max_bytes=1 --param twoshot_bytes_per_cta=2048" "ll2_max_bytes=1 --param twoshot_bytes_per_cta=16384" "ll2_max_bytes=1 --param max_ctas=74"; do
i=$((i+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+i)) bench.py --gpus $n --mode sweep --sweep-min 262144 --sweep-max 33554432 --algos ring_rsa --param $prm --out gpurun_out/t2/s_${n}_$i.csv > gpurun_out/t2/s_${n}_$i.out 2>gpurun_out/t2/s_${n}_$i.err
echo "$n $i $prm rc=$?"
done; done
