python scripts/ab_dp.py c3 comb
python scripts/ab_dp.py c2 comb
timeout 900 python -m pytest tests/test_decode_pass_gpu.py tests/test_full_shape_gpu.py tests/test_offload_gpu.py -x -q 2>&1 | tail -4
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; tail -2 gpurun_out/r2_bench2.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_pass -s 3 -c 1 -o gpurun_out/r2_dp_little python scripts/prof_dp2.py c3 little 512 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches2.csv python bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline --no-ep > /dev/null 2>&1
bash scripts/gpu/sanitize.sh
