set -x
mkdir -p gpurun_out
for i in 1 2; do
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1_$i.jsonl 2>/dev/null; python -c "import sys,json; d=json.loads(open('gpurun_out/bench_c1_$i.jsonl').read().strip().splitlines()[-1]); b=d['build']; print(d['value'], d['ms_per_step'], b['seconds'], b['points_per_s'], b['phases_ms'], b['roofline']['frac'])"
done
