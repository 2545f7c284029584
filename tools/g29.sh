# round-2 closing run A: the new parity tests (C4 vs the library-LP oracle, C2 samples vs both
# oracles), then the C1 / C3 / C4 bench lines (a timed line per decode config)
mkdir -p gpurun_out
TAG=${TAG:-g29}
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider --durations=8 -k "config4 or config2_sample" > gpurun_out/gpu_tests_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
timeout 600 python bench.py --config 1 --frames 16384 --step-systems 0 > gpurun_out/bench_c1_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_c1_$TAG.log
timeout 900 python bench.py --config 3 --frames 8192 --step-systems 0 > gpurun_out/bench_c3_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_c3_$TAG.log
timeout 1500 python bench.py --config 4 --frames ${C4F:-592} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --step-systems 0 > gpurun_out/bench_c4_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_c4_$TAG.log
