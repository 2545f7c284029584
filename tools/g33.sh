# A/B: cached PCG-window offsets (v2) and static-shared phase clocks on top (v3) vs the default build;
# parity subset run against the v3 library
mkdir -p gpurun_out
TAG=${TAG:-g33}
LIBS="libalp.so libalp_v2.so libalp_v3.so libalp.so libalp_v2.so libalp_v3.so" TAG=$TAG bash tools/gpu_ab.sh
for L in libalp.so libalp_v3.so libalp.so libalp_v3.so; do
  echo "== C5 $L" >> gpurun_out/ab_$TAG.log
  ALP_LIB=paper_0902_0657_b200/$L timeout 600 python bench.py --frames 148 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --snr-sweep 0 --step-systems 65536 2>&1 | python -c "
import sys, json
for ln in sys.stdin:
    if ln.startswith('{'):
        d = json.loads(ln); s = d['step_solve']; print({k: s[k] for k in ('systems_per_s', 'ms_per_call', 'pcg_iters_per_s', 'status_counts')})
    elif ln.strip(): print(ln.rstrip())
" >> gpurun_out/ab_$TAG.log 2>&1
done
ALP_LIB=paper_0902_0657_b200/libalp_v3.so timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "not rowwise_mts_matches and not config4" > gpurun_out/gpu_tests_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
