timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
tail -3 gpurun_out/r2_bench1.err
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/r2_gputest2.log
cat gpurun_out/r2_gputest2.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_pass -s 2 -c 1 -o gpurun_out/r2_dp1 python scripts/prof_dp.py c3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline > /dev/null 2>&1
python -c "import json; d=json.load(open('gpurun_out/r2_bench1.json')); print(d['value'], d['speedup_vs_full_topk'], d['roofline']['frac'], json.dumps(d['configs'])[:3000])"
