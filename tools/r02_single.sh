#!/bin/bash
# round-2 single-GPU evidence pass: sanitizer summaries, ncu of the virtual
# headline kernel (p = 4, 8), N=1 bench line and its kernel launch list
mkdir -p gpurun_out
timeout 600 python tools/sanitize_virtual.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_virtual.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.log
done
for p in 4 8; do
  timeout 300 python tools/virtual_agg.py --p $p > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:collective_kernel -s 2 -c 1 \
    -o gpurun_out/r02_virtual_agg_p$p -f python tools/virtual_agg.py --p $p > gpurun_out/ncu_virtual_p$p.log 2>&1
  echo "ncu p=$p rc=$?"
  ncu -i gpurun_out/r02_virtual_agg_p$p.ncu-rep --page raw --csv > gpurun_out/r02_virtual_agg_p${p}_raw.csv 2>/dev/null
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_n1.json 2> gpurun_out/r02_bench_n1.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "launch list rc=$?"
