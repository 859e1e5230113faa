timeout 1500 python -m pytest tests/test_kernels_gpu.py -k attn_decode -x -q 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_decode_pass_gpu.py tests/test_runtime_gpu.py tests/test_full_shape_gpu.py tests/test_decode_gpu.py tests/test_offload_gpu.py -x -q 2>&1 | tail -4
python scripts/ab_dp.py c5 gqa
