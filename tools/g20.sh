mkdir -p gpurun_out
timeout 900 python tools/c5_eval.py > gpurun_out/c5eval.log 2>&1
CFGS="4:0" F=16384 timeout 300 python tools/tune_smem.py > gpurun_out/tune20.log 2>&1
ALP_SM_D2=1 CFGS="4:0" F=16384 timeout 300 python tools/tune_smem.py >> gpurun_out/tune20.log 2>&1
