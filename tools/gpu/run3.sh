set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err; tail -3 gpurun_out/bench_c1.err
ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/search_c1_L1024 python tools/ab_search.py --L 1024 --profile > gpurun_out/ncu_1024.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/search_c1_L200 python tools/ab_search.py --L 200 --profile > gpurun_out/ncu_200.log 2>&1
tail -2 gpurun_out/ncu_1024.log gpurun_out/ncu_200.log
