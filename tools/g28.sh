# batched Alg. 7 peel v2: pivot / decode parity subset, A/B cycles vs the sequential peel, batch counts
mkdir -p gpurun_out
TAG=${TAG:-g28}
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider -k "${TESTK:-step or config1 or config2_sample or h7 or config3}" > gpurun_out/gpu_tests_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
LIBS="libalp.so libalp_seq.so" TAG=$TAG bash tools/gpu_ab.sh
ALP_LIB=paper_0902_0657_b200/libalp_count.so timeout 200 python tools/peel_diag.py >> gpurun_out/ab_$TAG.log 2>&1
