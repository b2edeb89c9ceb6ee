set -x
mkdir -p gpurun_out
for i in 1 2 3; do
python bench.py --steps 5 --warmup 3 --no-cpu --no-build-roofline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); b=d['build']; print(b['seconds'], b['points_per_s'], b['phases_ms'])"
done
