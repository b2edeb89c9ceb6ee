set -x
mkdir -p gpurun_out
python tools/ab_search.py --L 512,832,1024 --var GANN_GTAB_MIN_L=0,384 --rounds 2 > gpurun_out/ab_gtab.log 2>&1; grep -E "MQPS" gpurun_out/ab_gtab.log
python -m pytest tests/test_gpu_baseline.py tests/test_gpu_search.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -2 gpurun_out/t_s.log
