#!/bin/bash
# GPU-box script: GPU suite, default bench line, then the profile captures of tools/g25.sh.
# TAG names the captures; SKIP_TESTS=1 / SKIP_BENCH=1 / SKIP_PROF=1 skip a stage.
mkdir -p gpurun_out
TAG=${TAG:-r2x}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m "${TESTM:-gpu}" -q --durations=15 --timeout 900 -p no:cacheprovider -k "${TESTK:-}" > gpurun_out/gpu_tests_$TAG.log 2>&1
  echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 1200 python bench.py ${BENCH:-} > gpurun_out/bench_$TAG.log 2>&1
  echo "bench exit $?" >> gpurun_out/bench_$TAG.log
fi
if [ -z "$SKIP_PROF" ]; then
  TAG=$TAG bash tools/g25.sh
fi
