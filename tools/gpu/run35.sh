set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_search.py tests/test_gpu_baseline.py tests/test_gpu_build.py tests/test_gpu_checked.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -15 gpurun_out/t_s.log
python tools/ab_search.py --L 64,128,200,832 --rounds 2 --var GANN_BATCH_EB=0,4,8 > gpurun_out/ab_batch.log 2>&1; grep -E "MQPS|diag|Error|error|assert" gpurun_out/ab_batch.log
