timeout 300 python -m pytest tests/test_gpu_virtual.py -x -q -k "single_rank" 2>&1 | tail -2
HOST=1 timeout 200 python tools/timeline.py 2>&1 | grep -v "^W1\|Warn\|warn" | head -60
