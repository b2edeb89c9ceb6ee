set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_batch.py tests/test_gpu_checked.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -3 gpurun_out/t_s.log
python tools/ab_search.py --L 400,832 --rounds 2 --reps 5 --var GANN_GTAB_WIDE=0,1 > gpurun_out/ab_a.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_a.log
python tools/ab_search.py --config c4 --n 100000000 --L 400,832 --rounds 1 --reps 3 --var GANN_BATCH_EB=0,4 > gpurun_out/ab_100M.log 2>&1; grep -E "MQPS|Error|error|assert|build_ms" gpurun_out/ab_100M.log
