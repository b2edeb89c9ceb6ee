set -x
mkdir -p gpurun_out
GANN_BATCH_CARVE=100 ncu --section WarpStateStats --section SourceCounters --section MemoryWorkloadAnalysis --section Occupancy --section SchedulerStats --clock-control none --profile-from-start off -c 1 -o gpurun_out/batch_carve100 python tools/ab_search.py --L 832 --profile > gpurun_out/ncu_c100.log 2>&1; tail -2 gpurun_out/ncu_c100.log
ncu -i gpurun_out/batch_carve100.ncu-rep --page details > gpurun_out/carve100_details.txt 2>&1
ncu -i gpurun_out/batch_carve100.ncu-rep --page raw --csv > gpurun_out/carve100_raw.csv 2>&1
