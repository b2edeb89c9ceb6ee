set -x
mkdir -p gpurun_out
GANN_LIB=libgann_base.so python tools/ab_search.py --L 200,832 --rounds 2 > gpurun_out/ab_base.log 2>&1; grep -E "MQPS" gpurun_out/ab_base.log
python tools/ab_search.py --L 200 --var GANN_SEARCH_NEXTPF=0,1 --rounds 2 > gpurun_out/ab_200.log 2>&1; grep -E "MQPS" gpurun_out/ab_200.log
python tools/ab_search.py --L 832 --var GANN_SEARCH_NEXTPF=0,1 --var GANN_GTAB_KEEP=0,1 --var GANN_GTAB_LOG2=11,12 --rounds 2 > gpurun_out/ab_832.log 2>&1; grep -E "MQPS" gpurun_out/ab_832.log
for keep in 0 1; do
GANN_GTAB_KEEP=$keep ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none --profile-from-start off -c 1 python tools/ab_search.py --L 832 --profile > gpurun_out/ncu_keep$keep.log 2>&1; grep -E "dram__|gpu__time|hit_rate" gpurun_out/ncu_keep$keep.log
done
