set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1; tail -2 gpurun_out/t_gpu.log
GANN_BATCH_DEBUG=1 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err; grep "search launch: L" gpurun_out/bench_c1.err | sort | uniq -c | sort -k5n | awk '{print $5,$8,$9,$10,$11}' | uniq | tr '\n' ';'
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_c1.jsonl').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['at_sweep_end']['frac'], d['e2e']['value'], d['build']['points_per_s'], d['parity']['graph_sha256'], d['parity']['ids_sha256'])
print([(c['L'], c['ms_per_launch']) for c in d['qps_curve']['sweep'] if c['L'] in (10,64,128,200)])
PY
python tools/ab_search.py --L 64,128,200 --rounds 2 --reps 5 2>&1 | grep MQPS
