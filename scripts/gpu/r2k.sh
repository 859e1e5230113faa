for i in 1 2; do
python scripts/ab_dp.py c3 cur
MOBILE_LIB=paper_2510_12357_b200/variants/libmobile_head.so python scripts/ab_dp.py c3 head
done
python scripts/ab_dp.py c2 cur
MOBILE_LIB=paper_2510_12357_b200/variants/libmobile_head.so python scripts/ab_dp.py c2 head
timeout 900 python -m pytest tests/test_decode_pass_gpu.py tests/test_full_shape_gpu.py -x -q 2>&1 | tail -3
python scripts/trace_dp.py c3 little > gpurun_out/r2_trace_ll2.json
python -c "import json;d=json.load(open('gpurun_out/r2_trace_ll2.json'));print(json.dumps(d['per_kind']))"
