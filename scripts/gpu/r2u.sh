for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-configs --no-ep --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('persistent-zs', d['value'], d['baseline_full_topk']['value'], d['speedup_vs_full_topk'], d['pcie']['frac'])"
MOBILE_PERSISTENT=0 python bench.py --steps 20 --warmup 5 --no-configs --no-ep --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('per-op-seg', d['value'], d['baseline_full_topk']['value'], d['speedup_vs_full_topk'], d['pcie']['frac'])"
done
