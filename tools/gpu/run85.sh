set -x
mkdir -p gpurun_out
for i in 1 2 3; do
GANN_TRACE_START=1 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c1_$i.jsonl 2> gpurun_out/bench_c1_$i.err; grep "build start phase" gpurun_out/bench_c1_$i.err | head -2; python -c "import sys,json; d=json.loads(open('gpurun_out/bench_c1_$i.jsonl').read().strip().splitlines()[-1]); b=d['build']; print(b['seconds'], b['phases_ms']['start'])"
done
