#!/bin/bash
# GPU-box script: launch plan, GPU suite (TESTK filter), smoke, a short C2 3.0 dB bench line and
# the per-phase cycle breakdown (tools/tune_smem.py).  TAG names the outputs.
mkdir -p gpurun_out
TAG=${TAG:-q}
python - > gpurun_out/plan_$TAG.txt 2>&1 <<'PY'
import paper_0902_0657_b200 as alp
from synth import config_code
for cfg in (1, 2, 3, 5):
    c = alp.Code.from_synth(config_code(cfg))
    print(cfg, "decode", alp.launch_info(c, 16384), "step", alp.launch_info(c, 65536, step=True))
PY
if [ -z "$SKIP_TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m "${TESTM:-gpu}" -x -q --durations=10 --timeout 900 -p no:cacheprovider -k "${TESTK:-}" > gpurun_out/gpu_tests_$TAG.log 2>&1
  echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1
fi
timeout 900 python bench.py --steps 3 --warmup 3 --snr-sweep 0 --no-cpu-baseline ${BENCH:-} > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
F=4096 CFGS=${CFGS:-0:0} timeout 600 python tools/tune_smem.py > gpurun_out/tune_$TAG.log 2>&1
if [ -n "$TAIL" ]; then
  F=${TAILF:-4096} timeout 900 python tools/tail_stats.py > gpurun_out/tail_$TAG.log 2>&1
fi
