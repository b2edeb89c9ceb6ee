set -x
mkdir -p gpurun_out
for w in 4 2 1; do
GANN_BATCH_WPB=$w GANN_BATCH_DEBUG=1 python bench.py --steps 20 --warmup 5 --no-cpu --no-build-roofline > gpurun_out/bench_w$w.jsonl 2> gpurun_out/bench_w$w.err
grep "batch launch: L 832" gpurun_out/bench_w$w.err | sort | uniq -c | tail -2
python - <<PY
import json
d=json.loads(open('gpurun_out/bench_w$w.jsonl').read().strip().splitlines()[-1])
print($w, d['value'], d['ms_per_step'], d['roofline']['launch_event_span_ms_mean'], d['e2e']['value'], d['e2e']['blocking']['value'])
PY
done
