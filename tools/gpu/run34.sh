set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1; tail -5 gpurun_out/t_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err; tail -3 gpurun_out/bench_c1.err
python tools/ab_search.py --L 200,832 --rounds 2 --var GANN_SEARCH_DIAG=0,1 > gpurun_out/ab_diag.log 2>&1; grep -E "MQPS|diag" gpurun_out/ab_diag.log
