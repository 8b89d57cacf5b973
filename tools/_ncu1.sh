set -e
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-check"
$B > gpurun_out/ncu_plain.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_bench_n1.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:batched_copy -s 6 -c 1 -o /tmp/pack $B > /dev/null 2>&1
ncu -i /tmp/pack.ncu-rep --page raw --csv > gpurun_out/ncu_pack_raw.csv
ncu -i /tmp/pack.ncu-rep --page details --csv > gpurun_out/ncu_pack_details.csv
V="python tools/virtual_ar.py --p 4 --n 16320000 --algo ring_rsa --iters 3"
$V
ncu --set full --clock-control none --import-source on -k regex:collective_kernel -s 1 -c 1 -o /tmp/coll $V > /dev/null 2>&1
ncu -i /tmp/coll.ncu-rep --page raw --csv > gpurun_out/ncu_coll_raw.csv
ncu -i /tmp/coll.ncu-rep --page details --csv > gpurun_out/ncu_coll_details.csv
echo done
