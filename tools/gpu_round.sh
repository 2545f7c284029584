#!/bin/bash
# GPU-box script: GPU tests, then a short bench run (outputs under gpurun_out/).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import paper_0902_0657_b200 as a; print(a.lib().alp_build_info())" > gpurun_out/lib.txt 2>&1
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m "${TESTM:-gpu}" -q --durations=15 --timeout 900 -p no:cacheprovider -k "${TESTK:-}" > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests.log
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py $BENCH > gpurun_out/bench.log 2>&1
  echo "bench exit $?" >> gpurun_out/bench.log
fi
