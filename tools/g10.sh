mkdir -p gpurun_out
for v in scratch/variants/libalp_noassume.so paper_0902_0657_b200/libalp.so; do
  echo "== $v" >> gpurun_out/dbg10.log
  ALP_LIB=$v STEP=1 NF=4 timeout 120 python tools/memcheck_c1.py >> gpurun_out/dbg10.log 2>&1; echo "exit $?" >> gpurun_out/dbg10.log
  ALP_LIB=$v STEP=0 NF=4 CFG=2 timeout 120 python tools/memcheck_c1.py >> gpurun_out/dbg10.log 2>&1; echo "exit $?" >> gpurun_out/dbg10.log
done
