mkdir -p gpurun_out
for v in scratch/variants/scalar.so; do
  echo "== $v" >> gpurun_out/tune17.log
  ALP_LIB=$v CFGS="4:0" F=16384 timeout 300 python tools/tune_smem.py >> gpurun_out/tune17.log 2>&1
done
TAG=r2c PFRAMES=1184 bash tools/g6.sh
