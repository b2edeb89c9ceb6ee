set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err; tail -2 gpurun_out/bench_c1.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_c1.jsonl 2> gpurun_out/bench_ref_c1.err; tail -2 gpurun_out/bench_ref_c1.err
