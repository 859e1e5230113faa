for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-configs --no-ep --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['value'], d['mobile']['wall_ms_per_step'], d['pcie']['frac'], d['speedup_vs_full_topk'])"
MOBILE_DP_PF_KB=0 python bench.py --steps 20 --warmup 5 --no-configs --no-ep --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pf0', d['value'], d['mobile']['wall_ms_per_step'], d['pcie']['frac'], d['speedup_vs_full_topk'])"
done
timeout 900 python -m pytest tests/test_ep_engine_gpu.py tests/test_ep_p2p_gpu.py tests/test_ep_gpu.py -x -q 2>&1 | tail -15
