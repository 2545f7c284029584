mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "golden_step or partial or float or first_ipm or plain_cg_option or empty or config1 or h1 or h7 or ragged or config3 or certificate_needs or shards" > gpurun_out/t8.log 2>&1; echo "pytest exit $?" >> gpurun_out/t8.log
CFGS="4:0,2:0,3:0,4:8" F=16384 timeout 900 python tools/tune_smem.py > gpurun_out/tune8.log 2>&1
