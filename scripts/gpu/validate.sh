timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/r2_gputest6.log; cat gpurun_out/r2_gputest6.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench5.json 2> gpurun_out/r2_bench5.err; tail -2 gpurun_out/r2_bench5.err
python -c "import json; d=json.load(open('gpurun_out/r2_bench5.json')); print(d['value'], d['speedup_vs_full_topk'], d['roofline']['frac'], d['pcie']['frac']); c=d['configs']; print(json.dumps({k: (v['decode'] if 'decode' in v else v) for k,v in c.items()})[:2500]); print(json.dumps(c['c5'].get('prefill'))); print(json.dumps(d['ep']))"
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/r2_bench_ref.json; cat gpurun_out/r2_bench_ref.json | cut -c1-300
