mkdir -p gpurun_out
NF=1 timeout 900 python tools/diag_c4.py > gpurun_out/c4.log 2>&1; echo "c4 exit $?" >> gpurun_out/c4.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 -k "not config4" > gpurun_out/t5.log 2>&1; echo "pytest exit $?" >> gpurun_out/t5.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.log 2>&1
