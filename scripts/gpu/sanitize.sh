# compute-sanitizer over the small-shape -m gpu tests (full-shape tests stream
# GBs per launch and are out of reach under instrumentation)
S=/usr/local/cuda/bin/compute-sanitizer
SEL="tests/test_kernels_gpu.py tests/test_grouped_gemm_gpu.py tests/test_decode_pass_gpu.py::test_persistent_matches_oracle tests/test_runtime_gpu.py tests/test_ep_p2p_gpu.py::test_p2p_ep_world1"
timeout 2400 $S --tool memcheck --target-processes all --print-limit 20 --error-exitcode 0 python -m pytest $SEL -x -q -k "not qwen_full_size" -p no:cacheprovider > gpurun_out/r2_memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r2_memcheck.log | tail -5
timeout 1800 $S --tool racecheck --racecheck-report hazard --print-limit 20 --error-exitcode 0 python -m pytest tests/test_kernels_gpu.py tests/test_decode_pass_gpu.py::test_persistent_matches_oracle -x -q -k "not qwen_full_size" -p no:cacheprovider > gpurun_out/r2_racecheck.log 2>&1
echo "racecheck rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/r2_racecheck.log | tail -5
