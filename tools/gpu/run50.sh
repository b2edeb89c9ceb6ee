set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_batch.py tests/test_gpu_baseline.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -3 gpurun_out/t_s.log
python tools/ab_search.py --L 400,832,1280 --rounds 2 --reps 5 --var GANN_SEARCH_NEXTPF=0,1 > gpurun_out/ab_a.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_a.log
