# round-2 closing run: full GPU suite, smoke, default bench line, C3 / C4 bench lines, ncu captures
# (launch list + full capture of the C2 3.0 dB decode and of the config-5 step kernel; a
# section-limited capture of a C2 2.0 dB decode, whose straggler frames make --set full's ~40
# replays of a 20 s kernel impractical)
mkdir -p gpurun_out
TAG=${TAG:-r2z}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=15 --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 600 python bench.py --config 1 --frames 16384 --step-systems 0 > gpurun_out/bench_c1_$TAG.log 2>&1
timeout 900 python bench.py --config 3 --frames 8192 --step-systems 0 > gpurun_out/bench_c3_$TAG.log 2>&1
CMD="python bench.py --frames 1184 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --snr-sweep 0 --step-systems 0"
CMD2="python bench.py --frames 296 --snr-idx 0 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --snr-sweep 0 --step-systems 0"
CMD5="python bench.py --frames 148 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --snr-sweep 0 --step-systems 16384"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && $CMD5 > gpurun_out/prof_plain5_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:alp_decode_kernel -s 1 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:pcg_step_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG}_c5 $CMD5 > gpurun_out/ncu_full5_$TAG.log 2>&1
echo "profile exit $?" >> gpurun_out/prof_plain_$TAG.log
$CMD2 > gpurun_out/prof_plain2_$TAG.log 2>&1 &&
timeout 900 ncu --section SpeedOfLight --section WarpStateStats --section MemoryWorkloadAnalysis --section Occupancy --section LaunchStats --clock-control none -k regex:alp_decode_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG}_2db $CMD2 > gpurun_out/ncu_2db_$TAG.log 2>&1
echo "2 dB profile exit $?" >> gpurun_out/prof_plain2_$TAG.log
timeout 1500 python bench.py --config 4 --frames ${C4F:-1184} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --step-systems 0 > gpurun_out/bench_c4_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_c4_$TAG.log
