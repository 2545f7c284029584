mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -m gpu -q -p no:cacheprovider -k "c5_first or plain_cg or partial or float" > gpurun_out/t3.log 2>&1; echo "pytest exit $?" >> gpurun_out/t3.log
for cfg in "paper_0902_0657_b200/libalp.so 4:11,4:8,4:16,2:11" "scratch/variants/libalp_minb3.so 4:12,4:16,4:20" "scratch/variants/libalp_minb4.so 4:16,4:20,4:24"; do
  set -- $cfg
  echo "== $1" >> gpurun_out/tune3.log
  ALP_LIB=$1 CFGS=$2 F=4096 timeout 300 python tools/tune_smem.py >> gpurun_out/tune3.log 2>&1
done
