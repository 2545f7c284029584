mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -v -p no:cacheprovider --durations=15 -k "not config4" > gpurun_out/t19.log 2>&1; echo "pytest exit $?" >> gpurun_out/t19.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench19.log 2>&1; echo "bench exit $?" >> gpurun_out/bench19.log
K=80 timeout 900 python tools/e5_traces.py > gpurun_out/e5_19.log 2>&1
timeout 900 python tools/iteration_stats.py > gpurun_out/stats19.log 2>&1
