mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_decode.py -m gpu -q -x -k "golden or partial or float_ties or first_ipm or config1_all or h1 or h7 or ragged" -p no:cacheprovider > gpurun_out/t2.log 2>&1; echo "pytest exit $?" >> gpurun_out/t2.log
VARIANTS='[{}, {"pcg_forcing": 0.0}, {"pcg_max_iter": 300}, {"basis_correction": 0}]' timeout 900 python tools/diag_hard.py > gpurun_out/diag_hard.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --snr-sweep 0 --step-systems 0 > gpurun_out/bench2.log 2>&1
