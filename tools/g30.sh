# A/B: graph reads as LDS in sm mode (libalp.so) vs generic loads (libalp_base.so); parity subset
mkdir -p gpurun_out
TAG=${TAG:-g30}
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "${TESTK:-config1 or config2_sample or h7 or h1 or tie or equal_weights or ragged}" > gpurun_out/gpu_tests_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
LIBS="${LIBS:-libalp_base.so libalp.so libalp_base.so libalp.so}" TAG=$TAG bash tools/gpu_ab.sh
# config-5 step solve: gs instance (staged graph by LDS) vs the base library
for L in libalp_base.so libalp.so; do
  echo "== $L" >> gpurun_out/c5_$TAG.log
  ALP_LIB=paper_0902_0657_b200/$L timeout 600 python bench.py --frames 148 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --snr-sweep 0 --step-systems 65536 2>&1 | python -c "
import sys, json
for ln in sys.stdin:
    if ln.startswith('{'):
        d = json.loads(ln); s = d['step_solve']; print({k: s[k] for k in ('systems_per_s', 'ms_per_call', 'pcg_iters_per_s', 'status_counts')})
    elif ln.strip(): print(ln.rstrip())
" >> gpurun_out/c5_$TAG.log 2>&1
done
