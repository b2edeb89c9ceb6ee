set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err; tail -3 gpurun_out/bench_c1.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_c1.jsonl').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['at_sweep_end'], d['e2e'])
PY
python bench.py --config c0 --steps 20 --warmup 5 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['kernel'], d['roofline']['at_sweep_end'])"
