set -x
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:prune_prep_kernel --launch-skip 450 -c 1 -o gpurun_out/prep_mid python tools/bench_build.py --reps 1 > gpurun_out/ncu_prep.log 2>&1; tail -2 gpurun_out/ncu_prep.log
