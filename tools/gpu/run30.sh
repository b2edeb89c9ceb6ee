set -x
mkdir -p gpurun_out
for lib in libgann_mb6.so libgann_b200.so; do
GANN_LIB=$lib python tools/ab_search.py --L 640,832,1024 --var GANN_GTAB_NO_BAND=0,1 --rounds 2 > gpurun_out/ab_$lib.log 2>&1; grep -E "MQPS|diag" gpurun_out/ab_$lib.log
done
python -m pytest tests/test_gpu_baseline.py tests/test_gpu_search.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -2 gpurun_out/t_s.log
