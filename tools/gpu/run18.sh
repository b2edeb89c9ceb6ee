set -x
python -m pytest tests/test_gpu_baseline.py tests/test_gpu_search.py tests/test_gpu_checked.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -2 gpurun_out/t_s.log
GANN_LIB=libgann_b200.so python tools/bench_build.py --reps 2 > gpurun_out/bb_new.log 2>&1; grep -E "build 1" gpurun_out/bb_new.log
GANN_LIB=libgann_b200.so python tools/ab_search.py --L 128,200,832 --rounds 2 > gpurun_out/ab_new.log 2>&1; grep -E "MQPS" gpurun_out/ab_new.log
