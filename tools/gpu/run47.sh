set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1; tail -8 gpurun_out/t_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err; tail -3 gpurun_out/bench_c1.err; python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_c1.jsonl').read().strip().splitlines()[-1])
print({k:d[k] for k in ('value','ms_per_step')}, d['config']['L_search'], d['roofline']['frac'], d['e2e']['value'], d['build']['points_per_s'], d['parity'])
PY
