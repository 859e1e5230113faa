set -x
MOBILE_DP_PF_KB=-1 python scripts/ab_dp.py c3 newcons
MOBILE_DP_PF_KB=-1 python scripts/ab_dp.py c2 newcons
MOBILE_DP_PF_KB=-1 timeout 600 python -m pytest tests/test_decode_pass_gpu.py tests/test_full_shape_gpu.py tests/test_kernels_gpu.py -x -q 2>&1 | tail -5
MOBILE_DP_PF_KB=-1 python scripts/trace_dp.py c3 little > gpurun_out/r2_trace_little2.json
MOBILE_DP_PF_KB=-1 python scripts/events_dp.py 0 77 > gpurun_out/r2_events2.txt
