set -x
for s in 2 3 4; do
python bench.py --steps 24 --warmup 6 --streams $s --no-cpu --no-build-roofline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($s, d['value'], d['ms_per_step'], d['e2e']['value'])"
done
