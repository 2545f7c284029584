# A/B: gs instance with LDS window + sign tables (libalp.so) vs the previous build (libalp_g1.so) on
# config 5; config 3 with the graph staged in shared memory (ALP_GRAPH_MAX_KB=72) vs global
mkdir -p gpurun_out
TAG=${TAG:-g31}
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "${TESTK:-c5_first_1024 or plain_cg_option or tie or equal_weights or config3 or incremental}" > gpurun_out/gpu_tests_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
run5() {
  timeout 600 python bench.py --frames 148 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --snr-sweep 0 --step-systems 65536 2>&1 | python -c "
import sys, json
for ln in sys.stdin:
    if ln.startswith('{'):
        d = json.loads(ln); s = d['step_solve']; print({k: s[k] for k in ('systems_per_s', 'ms_per_call', 'pcg_iters_per_s', 'status_counts')})
    elif ln.strip(): print(ln.rstrip())
"
}
run3() {
  timeout 600 python bench.py --config 3 --frames 2368 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --step-systems 0 2>&1 | python -c "
import sys, json
for ln in sys.stdin:
    if ln.startswith('{'):
        d = json.loads(ln); print(round(d['value'], 1), 'frames/s', d['launch'], {k: round(v, 3) for k, v in d['pcg_phase']['shares'].items()})
    elif ln.strip(): print(ln.rstrip())
"
}
for L in libalp_g1.so libalp.so libalp_g1.so libalp.so; do
  echo "== C5 $L" >> gpurun_out/ab_$TAG.log
  ALP_LIB=paper_0902_0657_b200/$L run5 >> gpurun_out/ab_$TAG.log 2>&1
done
for KB in 48 72 48 72; do
  echo "== C3 graph max $KB KB" >> gpurun_out/ab_$TAG.log
  ALP_GRAPH_MAX_KB=$KB run3 >> gpurun_out/ab_$TAG.log 2>&1
done
