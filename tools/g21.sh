mkdir -p gpurun_out
timeout 900 python tools/c5_eval.py > gpurun_out/c5eval.log 2>&1
CFGS="4:0" F=16384 timeout 300 python tools/tune_smem.py > gpurun_out/tune21.log 2>&1
NF=1184 timeout 1200 python tools/diag_c4.py > gpurun_out/c4_1184.log 2>&1
