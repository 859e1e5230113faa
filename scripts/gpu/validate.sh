# the full -m gpu suite, the default bench line, the reference arm, and the
# ncu launch list of a short bench run (outputs under gpurun_out/)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/r2_gputest.log; cat gpurun_out/r2_gputest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -2 gpurun_out/r2_bench.err
python -c "import json; d=json.load(open('gpurun_out/r2_bench.json')); print(d['value'], d['speedup_vs_full_topk'], d['roofline']['frac'], d['pcie']['frac']); c=d['configs']; print(json.dumps({k: (v['decode'] if 'decode' in v else v) for k,v in c.items()})[:2500]); print(json.dumps(c['c5'].get('prefill'))); print(json.dumps(d['ep']))"
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/r2_bench_ref.json; cut -c1-300 gpurun_out/r2_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline --no-ep > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/r2_bench_launches.csv > gpurun_out/r2_bench_launches_summary.txt; head -12 gpurun_out/r2_bench_launches_summary.txt
