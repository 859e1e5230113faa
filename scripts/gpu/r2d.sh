set -x
python scripts/ab_dp.py c3 mma
python scripts/ab_dp.py c2 mma
python scripts/ab_dp.py c5 mma
timeout 900 python -m pytest tests/test_decode_pass_gpu.py tests/test_full_shape_gpu.py tests/test_functional_gpu.py tests/test_offload_gpu.py -x -q 2>&1 | tail -5
python scripts/trace_dp.py c3 little > gpurun_out/r2_trace_little3.json
python scripts/events_dp.py 0 77 > gpurun_out/r2_events3.txt
