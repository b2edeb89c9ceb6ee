set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err; tail -2 gpurun_out/bench_c1.err
python bench.py --config c0 --steps 20 --warmup 5 > gpurun_out/bench_c0.jsonl 2> gpurun_out/bench_c0.err; tail -2 gpurun_out/bench_c0.err
python bench.py --impl reference --config c0 --steps 5 --warmup 2 > gpurun_out/bench_ref_c0.jsonl 2> gpurun_out/bench_ref_c0.err; tail -2 gpurun_out/bench_ref_c0.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
