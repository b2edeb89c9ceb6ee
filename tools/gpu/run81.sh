set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_batch.py tests/test_gpu_baseline.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -2 gpurun_out/t_s.log
for w in auto; do
if [ $w = auto ]; then unset GANN_BATCH_WPB; else export GANN_BATCH_WPB=$w; fi
GANN_BATCH_DEBUG=1 python bench.py --steps 20 --warmup 5 --no-cpu --no-build-roofline > gpurun_out/bench_w$w.jsonl 2> gpurun_out/bench_w$w.err; grep "batch launch" gpurun_out/bench_w$w.err | sort | uniq -c | sort -k5n | awk "{print \$5,\$6,\$10,\$11,\$12,\$13}" | uniq | tr "\n" ";"
python - <<PY
import json
d=json.loads(open('gpurun_out/bench_w$w.jsonl').read().strip().splitlines()[-1])
print('$w', d['value'], d['ms_per_step'], [(c['L'], c['ms_per_launch']) for c in d['qps_curve']['past_sweep']])
PY
done
