set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf -p no:cacheprovider -k "baseline or long_walks or repeated or invalid_rows or staged" > gpurun_out/t_new.log 2>&1; tail -5 gpurun_out/t_new.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err; tail -3 gpurun_out/bench_c1.err
GANN_LIB=libgann_base.so python tools/ab_search.py --L 200 --rounds 3 > gpurun_out/ab_base.log 2>&1
python tools/ab_search.py --L 200 --rounds 3 > gpurun_out/ab_new.log 2>&1
grep MQPS gpurun_out/ab_base.log gpurun_out/ab_new.log
python bench.py --config c0 --steps 20 --warmup 5 > gpurun_out/bench_c0.jsonl 2> gpurun_out/bench_c0.err
python bench.py --impl reference --config c0 --steps 5 --warmup 2 > gpurun_out/bench_ref_c0.jsonl 2> gpurun_out/bench_ref_c0.err
nproc; lscpu | grep "Model name"
