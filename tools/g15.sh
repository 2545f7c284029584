mkdir -p gpurun_out
for v in paper_0902_0657_b200/libalp.so scratch/variants/v1.so scratch/variants/v2.so scratch/variants/v3.so; do
  echo "== $v" >> gpurun_out/tune15.log
  ALP_LIB=$v CFGS="4:0" F=16384 timeout 300 python tools/tune_smem.py >> gpurun_out/tune15.log 2>&1
done
