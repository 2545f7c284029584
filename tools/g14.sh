mkdir -p gpurun_out
STEP=1 NF=4 timeout 120 python tools/memcheck_c1.py > gpurun_out/dbg14.log 2>&1; echo "exit $?" >> gpurun_out/dbg14.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "golden_step or partial or float or first_ipm or plain_cg_option or empty or config1 or h1 or h7 or ragged or config3 or certificate_needs" > gpurun_out/t14.log 2>&1; echo "pytest exit $?" >> gpurun_out/t14.log
CFGS="4:0,2:0" F=16384 timeout 900 python tools/tune_smem.py > gpurun_out/tune14.log 2>&1
