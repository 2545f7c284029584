mkdir -p gpurun_out
for v in paper_0902_0657_b200/libalp.so scratch/variants/sp42.so scratch/variants/sp44.so scratch/variants/sp24.so scratch/variants/sp84.so; do
  echo "== $v" >> gpurun_out/tune24.log
  ALP_LIB=$v CFGS="0:0" F=16384 timeout 300 python tools/tune_smem.py >> gpurun_out/tune24.log 2>&1
done
