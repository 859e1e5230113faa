timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/r2_gputest5.log; cat gpurun_out/r2_gputest5.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err; tail -2 gpurun_out/r2_bench4.err
python -c "import json; d=json.load(open('gpurun_out/r2_bench4.json')); print(d['value'], d['speedup_vs_full_topk'], d['roofline']['frac'], d['pcie']['frac'])"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
