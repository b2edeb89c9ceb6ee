set -x
for w in 4 2; do
GANN_SEARCH_WPB=$w python bench.py --steps 10 --warmup 3 --no-cpu --no-build-roofline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($w, d['build']['seconds'], [(c['L'], c['ms_per_launch']) for c in d['qps_curve']['sweep'] if c['L'] in (10,32,64,128,200)], [(c['L'], c['ms_per_launch']) for c in d['qps_curve']['past_sweep'] if c['L']<320])"
done
