set -x
mkdir -p gpurun_out
python tools/ab_search.py --L 640,832 --var GANN_SEARCH_PF2=0,1,2,4 --rounds 2 > gpurun_out/ab_pf2.log 2>&1; grep -E "MQPS" gpurun_out/ab_pf2.log
GANN_SEARCH_PF2=2 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none --profile-from-start off -c 1 python tools/ab_search.py --L 832 --profile > gpurun_out/ncu_pf2.log 2>&1; grep -E "dram__|gpu__time|hit_rate" gpurun_out/ncu_pf2.log
