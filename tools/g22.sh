mkdir -p gpurun_out
STEP=1 NF=4 timeout 120 python tools/memcheck_c1.py > gpurun_out/dbg22.log 2>&1; echo "exit $?" >> gpurun_out/dbg22.log
CFGS="0:0,4:0,5:0" F=16384 timeout 300 python tools/tune_smem.py > gpurun_out/tune22.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "config1 or h1 or h7 or ragged or golden_step or partial or float or first_ipm or c5_first" > gpurun_out/t22.log 2>&1; echo "pytest exit $?" >> gpurun_out/t22.log
