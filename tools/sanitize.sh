#!/bin/bash
# GPU-box script: compute-sanitizer memcheck / racecheck / synccheck on a tiny C1 decode + step
# solve, in the shared-memory window mode and the generic mode (smem_frames_per_sm = 8).
mkdir -p gpurun_out
TAG=${TAG:-san}
export NF=${NF:-3}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/memcheck_c1.py > gpurun_out/san_${tool}_sm_$TAG.log 2>&1
  echo "exit $?" >> gpurun_out/san_${tool}_sm_$TAG.log
  PRM="{'smem_frames_per_sm': 8}" timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/memcheck_c1.py > gpurun_out/san_${tool}_gm_$TAG.log 2>&1
  echo "exit $?" >> gpurun_out/san_${tool}_gm_$TAG.log
done
