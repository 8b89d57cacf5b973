#!/bin/bash
# N=1 headline A/B under knob settings (pack kernel): ab_n1.sh "k=v,k=v" ... ("-" = defaults)
for rep in 1 2; do
  for cfg in "$@"; do
    args=""
    [ "$cfg" != "-" ] && args=$(echo $cfg | tr ',' '\n' | sed 's/^/--param /' | tr '\n' ' ')
    python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu --no-virtual --no-check $args > gpurun_out/ab1.json 2>/dev/null
    python - "$cfg" "$rep" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab1.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(f"{sys.argv[1]:<30} rep={sys.argv[2]} ms/step={d['ms_per_step']} value={d['value']} pack_us={r['avg_launch_us']} frac={r['frac']}")
PY
  done
done
