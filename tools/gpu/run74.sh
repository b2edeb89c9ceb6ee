set -x
mkdir -p gpurun_out
for i in 1 2 3 4 5; do python -m pytest tests/test_gpu_batch.py tests/test_gpu_baseline.py tests/test_gpu_checked.py tests/test_gpu_partition.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1; done
for i in 1 2 3; do python tools/ab_search.py --L 832 --rounds 1 --reps 10 --var GANN_BATCH_EB=0,4 2>&1 | grep -E "MQPS|assert|Error"; done
