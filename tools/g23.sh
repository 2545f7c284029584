mkdir -p gpurun_out
CFGS="0:0" F=16384 timeout 300 python tools/tune_smem.py > gpurun_out/tune23.log 2>&1
