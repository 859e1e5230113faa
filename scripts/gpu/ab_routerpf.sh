mkdir -p gpurun_out
for m in c2 c5 c3; do for pf in 0 1; do MOBILE_ROUTER_PF=$pf timeout 300 python scripts/ab_perop.py $m pf$pf 2>&1 | tail -1; done; done > gpurun_out/r2_ab_routerpf.txt
cat gpurun_out/r2_ab_routerpf.txt
timeout 900 python -m pytest tests/test_ep_engine_gpu.py -q -x -k offloaded 2>&1 | tail -15 > gpurun_out/r2_ep_off.log; cat gpurun_out/r2_ep_off.log
MOBILE_ROUTER_PF=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_c5_perop.csv python scripts/prof_perop.py c5 > /dev/null 2>&1
python scripts/ncu_bw.py gpurun_out/r2_c5_perop.csv | head -20
