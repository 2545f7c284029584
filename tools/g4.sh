mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -m gpu -q -p no:cacheprovider -k "c5_first or plain_cg or partial or float or golden" > gpurun_out/t4.log 2>&1; echo "pytest exit $?" >> gpurun_out/t4.log
CFGS="4:8,2:8,2:7,2:6,1:6,1:5,3:7,4:6,2:5" F=4096 timeout 600 python tools/tune_smem.py > gpurun_out/tune4.log 2>&1
