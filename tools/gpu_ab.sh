#!/bin/bash
# GPU-box script: per-phase cycle breakdown (tools/tune_smem.py) of several library builds
# (LIBS = space-separated .so names under paper_0902_0657_b200/) and frames-per-CTA settings.
mkdir -p gpurun_out
TAG=${TAG:-ab}
for L in ${LIBS:-libalp.so}; do
  echo "== $L" >> gpurun_out/ab_$TAG.log
  ALP_LIB=paper_0902_0657_b200/$L F=${F:-4096} CFGS=${CFGS:-0:0} timeout 900 python tools/tune_smem.py >> gpurun_out/ab_$TAG.log 2>&1
done
