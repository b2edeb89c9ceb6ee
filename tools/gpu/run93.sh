set -x
for e in 4 3; do
GANN_BATCH_EB=$e python bench.py --steps 20 --warmup 5 --no-cpu --no-build-roofline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($e, d['value'], d['ms_per_step'])"
done
