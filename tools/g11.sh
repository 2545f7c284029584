mkdir -p gpurun_out
for v in paper_0902_0657_b200/libalp.so scratch/variants/libalp_sonly.so scratch/variants/libalp_aonly.so; do
  echo "== $v" >> gpurun_out/dbg11.log
  ALP_LIB=$v STEP=1 NF=4 timeout 120 python tools/memcheck_c1.py 2>&1 | grep -v "^ \|Traceback\|File\|Search\|CUDA kernel\|For debug\|Compile" >> gpurun_out/dbg11.log; echo "exit $?" >> gpurun_out/dbg11.log
done
