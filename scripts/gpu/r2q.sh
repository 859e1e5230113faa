timeout 600 python -m pytest tests/test_kernels_gpu.py -k attn_decode -x -q 2>&1 | tail -3
timeout 2000 python -m pytest tests/test_decode_pass_gpu.py tests/test_runtime_gpu.py tests/test_full_shape_gpu.py tests/test_decode_gpu.py tests/test_offload_gpu.py tests/test_functional_gpu.py tests/test_ep_engine_gpu.py -x -q 2>&1 | tail -5
python scripts/ab_dp.py c3 kvbf16
python scripts/ab_dp.py c5 kvbf16
