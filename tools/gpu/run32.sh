set -x
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 100 -c 1 -o gpurun_out/build_search_c1 python tools/bench_build.py --reps 1 > gpurun_out/ncu_bs.log 2>&1; tail -1 gpurun_out/ncu_bs.log
ncu --set full --import-source on --clock-control none -k regex:prune_prep_kernel --launch-skip 300 -c 1 -o gpurun_out/build_prep_c1 python tools/bench_build.py --reps 1 > gpurun_out/ncu_bp.log 2>&1; tail -1 gpurun_out/ncu_bp.log
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c1b.jsonl 2> gpurun_out/bench_c1b.err; tail -1 gpurun_out/bench_c1b.err
