python scripts/ab_dp.py c3 ll
python scripts/ab_dp.py c2 ll
python scripts/ab_dp.py c5 ll
timeout 1200 python -m pytest tests/test_decode_pass_gpu.py tests/test_full_shape_gpu.py tests/test_offload_gpu.py tests/test_runtime_gpu.py tests/test_functional_gpu.py -x -q 2>&1 | tail -4
python scripts/trace_dp.py c3 little > gpurun_out/r2_trace_ll.json
python -c "import json;d=json.load(open('gpurun_out/r2_trace_ll.json'));print(json.dumps(d['per_kind']))"
