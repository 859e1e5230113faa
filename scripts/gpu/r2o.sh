timeout 900 python -m pytest tests/test_ep_engine_gpu.py tests/test_ep_p2p_gpu.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 8 --warmup 3 --no-configs --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['ep']))"
