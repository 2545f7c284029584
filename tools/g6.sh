# plain run, then ncu launch list + one full capture of the decode kernel (C2 3.0 dB, 1184 frames)
mkdir -p gpurun_out
TAG=${TAG:-r2a}
CMD="python bench.py --frames ${PFRAMES:-1184} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --snr-sweep 0 --step-systems 0"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:alp_decode_kernel -s 1 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "profile exit $?" >> gpurun_out/prof_plain_$TAG.log

