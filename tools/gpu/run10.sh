set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1; tail -12 gpurun_out/t_gpu.log
GANN_SMALL_REPRUNE=0 python tools/bench_build.py --reps 2 > gpurun_out/bb0.log 2>&1; tail -1 gpurun_out/bb0.log
GANN_SMALL_REPRUNE=1 python tools/bench_build.py --reps 2 > gpurun_out/bb1.log 2>&1; tail -1 gpurun_out/bb1.log
ncu --set full --import-source on --clock-control none -k regex:reprune_small --launch-skip 50 -c 1 -o gpurun_out/reprune_small_c1b python tools/bench_build.py --reps 1 > gpurun_out/ncu_rs.log 2>&1; tail -1 gpurun_out/ncu_rs.log
