set -x
mkdir -p gpurun_out
for s in 2 3 4; do
python bench.py --steps 24 --warmup 6 --streams $s > gpurun_out/bench_s$s.jsonl 2> gpurun_out/bench_s$s.err
python - <<PY
import json
d=json.loads(open('gpurun_out/bench_s$s.jsonl').read().strip().splitlines()[-1])
print($s, {k:d[k] for k in ('value','ms_per_step')}, d['config']['L_search'], d['roofline']['frac'], d['e2e']['value'], d['build']['points_per_s'])
PY
done
