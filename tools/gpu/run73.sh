set -x
mkdir -p gpurun_out
for c in c2 c3; do
python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.jsonl 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err
python - <<PY
import json
d=json.loads(open('gpurun_out/bench_$c.jsonl').read().strip().splitlines()[-1])
print('$c', {k:d[k] for k in ('value','ms_per_step')}, d['config'].get('L_search'), d['config'].get('recall@10'), d['roofline']['frac'], d['e2e']['value'], d['build']['points_per_s'], d['cpu_baseline'].get('ids_identical_to_gpu'))
PY
done
