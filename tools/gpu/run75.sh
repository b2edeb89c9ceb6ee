set -x
mkdir -p gpurun_out
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c1.jsonl 2> gpurun_out/bench_ref_c1.err; tail -2 gpurun_out/bench_ref_c1.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_ref_c1.jsonl').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['config'], d['parity'], d['build'])
PY
