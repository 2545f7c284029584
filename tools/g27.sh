# batched Alg. 7 peel: pivot / decode parity subset, then A/B cycles vs the sequential peel
mkdir -p gpurun_out
TAG=${TAG:-g27}
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider -k "${TESTK:-step or config1 or config2_sample or h7 or config3}" > gpurun_out/gpu_tests_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
LIBS="libalp.so libalp_seq.so" TAG=$TAG bash tools/gpu_ab.sh
