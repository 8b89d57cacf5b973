timeout 600 python -m pytest tests/test_gpu_virtual.py -x -q -k "fuse or single_rank or aggregate or model" 2>&1 | tail -3
for b in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e --param bulk_copy=$b --steps 200 > gpurun_out/b1_$b.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b1_$b.json').read().strip().splitlines()[-1]); r=d['roofline']; print('bulk=$b', d['ms_per_step'], d['value'], r['achieved'], r['frac'], r['avg_launch_us'])"; done
python - <<'PY'
import torch
S=101_760_000//4
a=torch.randn(S,device="cuda"); b=torch.empty_like(a); fl=torch.empty(256<<20,dtype=torch.uint8,device="cuda")
ts=[]
for _ in range(50):
    fl.zero_(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ts=sorted(ts)[5:45]; m=sum(ts)/len(ts)
print("torch copy_ 101.76MB contiguous (L2 flushed): %.1f us  %.0f GB/s"%(m*1e3, 2*S*4/(m*1e-3)/1e9))
PY
