mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "golden_step or partial or float or first_ipm or plain_cg_option or empty or config1 or h1 or h7 or ragged or config3 or snr_idx2 or config2_sample and 2 or certificate_needs" > gpurun_out/t7.log 2>&1; echo "pytest exit $?" >> gpurun_out/t7.log
CFGS="4:8,4:7,4:11" F=16384 timeout 900 python tools/tune_smem.py > gpurun_out/tune7.log 2>&1
