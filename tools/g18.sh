mkdir -p gpurun_out
STEP=1 NF=4 timeout 120 python tools/memcheck_c1.py > gpurun_out/dbg18.log 2>&1; echo "exit $?" >> gpurun_out/dbg18.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "rowwise or thm5 or golden_step or partial or float or first_ipm or config1 or h1 or h7 or config3 or certificate_needs" > gpurun_out/t18.log 2>&1; echo "pytest exit $?" >> gpurun_out/t18.log
CFGS="4:0" F=16384 timeout 900 python tools/tune_smem.py > gpurun_out/tune18.log 2>&1
