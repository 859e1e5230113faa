set -x
python scripts/ab_dp.py c3 base
MOBILE_DP_PF_KB=-1 python scripts/ab_dp.py c3 nopf
MOBILE_DP_PF_KB=-1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:decode_pass -s 2 -c 1 python scripts/prof_dp.py c3 2>&1 | grep -E "dram__|gpu__time"
python scripts/trace_dp.py c3 little > gpurun_out/r2_trace_little.json
python scripts/events_dp.py 0 77 > gpurun_out/r2_events.txt
