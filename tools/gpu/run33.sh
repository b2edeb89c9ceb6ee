set -x
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:prune_prep_kernel --launch-skip 500 -c 6 -o gpurun_out/build_prep_c1b python tools/bench_build.py --reps 1 > gpurun_out/ncu_bp.log 2>&1; tail -1 gpurun_out/ncu_bp.log
ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 60 -c 4 -o gpurun_out/build_search_c1b python tools/bench_build.py --reps 1 > gpurun_out/ncu_bs.log 2>&1; tail -1 gpurun_out/ncu_bs.log
