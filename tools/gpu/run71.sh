set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-build-roofline > gpurun_out/ncu_bench.log 2>&1; tail -1 gpurun_out/ncu_bench.log | head -c 300
python tools/launch_summary.py gpurun_out/launches_bench.csv > gpurun_out/launches_bench.txt; head -12 gpurun_out/launches_bench.txt
grep -c "search_batch_kernel" gpurun_out/launches_bench.csv
