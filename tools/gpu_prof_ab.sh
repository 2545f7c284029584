#!/bin/bash
# GPU-box script: one ncu --set full capture of the decode kernel per library build (LIBS),
# C2 3.0 dB, F frames, through tools/tune_smem.py (after a plain run of the same command).
mkdir -p gpurun_out
TAG=${TAG:-pab}
for L in ${LIBS:-libalp.so}; do
  N=${L%.so}
  ALP_LIB=paper_0902_0657_b200/$L F=${F:-1184} CFGS=${CFGS:-0:0} timeout 600 python tools/tune_smem.py > gpurun_out/prof_${TAG}_$N.log 2>&1 &&
  ALP_LIB=paper_0902_0657_b200/$L F=${F:-1184} CFGS=${CFGS:-0:0} timeout 900 ncu --set full --clock-control none --import-source on -k regex:alp_decode_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG}_$N python tools/tune_smem.py >> gpurun_out/prof_${TAG}_$N.log 2>&1
  echo "exit $?" >> gpurun_out/prof_${TAG}_$N.log
done
