timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/r2_gputest4.log; cat gpurun_out/r2_gputest4.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err; tail -2 gpurun_out/r2_bench3.err
python -c "import json; d=json.load(open('gpurun_out/r2_bench3.json')); print(d['value'], d['speedup_vs_full_topk'], d['roofline']['frac'], d['pcie']['frac'], json.dumps(d['ep']))"
