set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err; tail -2 gpurun_out/bench_c1.err
python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err; tail -2 gpurun_out/bench_c2.err
python - <<'PY'
import json
for f in ('bench_c1','bench_c2'):
    d=json.loads(open(f'gpurun_out/{f}.jsonl').read().strip().splitlines()[-1])
    print(f, d['value'], d['ms_per_step'], d['config'].get('L_search'), d['config'].get('recall@10'), d['roofline']['frac'], d['e2e']['value'], d['build']['points_per_s'], d['parity']['graph_sha256'], d['parity']['ids_sha256'], d['cpu_baseline'].get('ids_identical_to_gpu'))
PY
