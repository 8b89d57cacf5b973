#!/bin/bash
# Device-side bounds-checked build (libcm_checked.so, -DCM_CHECKED) over the
# virtual tier, the fused-aggregate tests and the multi-process tier — the
# substitute for compute-sanitizer, which this GPU pool does not run.
export CM_LIB=$PWD/paper_1810_11112_b200/libcm_checked.so
mkdir -p gpurun_out
timeout 900 python tools/sanitize_virtual.py > gpurun_out/checked_workload.log 2>&1; echo "workload rc=$?"; tail -2 gpurun_out/checked_workload.log
timeout 1200 python -m pytest tests/test_gpu_fused_virtual.py tests/test_gpu_virtual.py tests/test_ps.py -m gpu -q -x \
  -k "not golden or c1" > gpurun_out/checked_virtual.log 2>&1; echo "virtual tests rc=$?"; tail -2 gpurun_out/checked_virtual.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k "sharing and 2 or sharing and 4" > gpurun_out/checked_mp.log 2>&1
echo "multi-process rc=$?"; tail -2 gpurun_out/checked_mp.log
grep -h "checked build" gpurun_out/checked_*.log | head -5
