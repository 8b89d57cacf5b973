#!/bin/bash
# Final-build evidence on one B200: N=1 launch list, ncu --set full of the N=1
# pack kernel and of the headline aggregate kernel on 4 virtual ranks.
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 600 $B > gpurun_out/r02f_bench_short.json 2>/dev/null; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02f_launches_bench_n1.csv $B > /dev/null 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batched_copy -s 6 -c 1 \
  -o gpurun_out/r02f_pack -f $B > /dev/null 2>&1; echo "ncu pack rc=$?"
ncu -i gpurun_out/r02f_pack.ncu-rep --page raw --csv > gpurun_out/r02f_pack_raw.csv 2>/dev/null
timeout 300 python tools/virtual_agg.py --p 4 > gpurun_out/r02f_virtual_agg.log 2>&1; echo "virtual rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collective_kernel -s 2 -c 1 \
  -o gpurun_out/r02f_virtual_agg_p4 -f python tools/virtual_agg.py --p 4 > /dev/null 2>&1; echo "ncu virtual rc=$?"
ncu -i gpurun_out/r02f_virtual_agg_p4.ncu-rep --page raw --csv > gpurun_out/r02f_virtual_agg_p4_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
