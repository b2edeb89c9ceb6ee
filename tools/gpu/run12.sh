set -x
mkdir -p gpurun_out
for lib in libgann_rb1.so libgann_b200.so libgann_rb8.so; do
  GANN_LIB=$lib python tools/ab_search.py --L 200,832 --rounds 2 > gpurun_out/ab_$lib.log 2>&1; grep -E "MQPS" gpurun_out/ab_$lib.log
done
GANN_LIB=libgann_b200.so python tools/ab_search.py --L 832 --var GANN_GTAB_MIN_L=0,384 --rounds 2 > gpurun_out/ab_gtab2.log 2>&1; grep MQPS gpurun_out/ab_gtab2.log
python -m pytest tests/test_gpu_baseline.py tests/test_gpu_search.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -2 gpurun_out/t_s.log
