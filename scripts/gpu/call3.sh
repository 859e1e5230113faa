mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ep_engine_gpu.py -q -x -k offloaded > gpurun_out/r2_ep_off.log 2>&1; tail -3 gpurun_out/r2_ep_off.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -2 gpurun_out/r2_bench.err
python -c "import json; d=json.load(open('gpurun_out/r2_bench.json')); print(d['value'], d['speedup_vs_full_topk'], d['roofline']['frac'], d['pcie']['frac'], d['clocks']); c=d['configs']; print({k: {b: (v['little']['ms'], v['full']['ms'], v['speedup_vs_full_topk']) for b, v in c[k]['decode'].items()} for k in ('c2','c4','c5')})"
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/r2_bench_ref.json; cut -c1-200 gpurun_out/r2_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline --no-ep > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/r2_bench_launches.csv > gpurun_out/r2_bench_launches_summary.txt; head -8 gpurun_out/r2_bench_launches_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_gemv -s 2 -c 2 -o gpurun_out/r2_sg_c5 -f python scripts/prof_perop.py c5 > gpurun_out/r2_sg_c5.log 2>&1; tail -2 gpurun_out/r2_sg_c5.log
