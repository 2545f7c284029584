# Round-2 final captures: C2 3.0 dB decode (plain run, launch list, ncu --set full), C5 step kernel
# (ncu --set full).  TAG names the outputs.
mkdir -p gpurun_out
TAG=${TAG:-r2f}
CMD="python bench.py --frames 1184 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --snr-sweep 0 --step-systems 0"
CMD5="python bench.py --frames 148 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --snr-sweep 0 --step-systems 16384"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 && $CMD5 > gpurun_out/prof_plain5_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:alp_decode_kernel -s 1 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:pcg_step_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG}_c5 $CMD5 > gpurun_out/ncu_full5_$TAG.log 2>&1
echo "profile exit $?" >> gpurun_out/prof_plain_$TAG.log
