set -x
mkdir -p gpurun_out
GANN_PRUNE_DEBUG=1 python tools/bench_build.py --reps 1 > gpurun_out/bb_d.log 2>&1; grep -E "re-prune lists" gpurun_out/bb_d.log | tail -2; grep build gpurun_out/bb_d.log | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_build.csv python tools/bench_build.py --reps 1 > gpurun_out/ncu_bb.log 2>&1
python tools/launch_summary.py gpurun_out/launches_build.csv | head -14
