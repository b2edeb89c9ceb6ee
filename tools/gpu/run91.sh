set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_batch.py tests/test_gpu_baseline.py tests/test_gpu_checked.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -2 gpurun_out/t_s.log
python tools/ab_search.py --nq 4000 --L 832,1024,2048,4096 --rounds 1 --reps 2 --var GANN_BATCH_EB=0,4 2>&1 | grep -E "MQPS|assert|Error|error"
