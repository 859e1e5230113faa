python scripts/ab_dp.py c3 hold
MOBILE_LIB=paper_2510_12357_b200/variants/libmobile_nohold.so python scripts/ab_dp.py c3 nohold
python scripts/ab_dp.py c2 hold
MOBILE_LIB=paper_2510_12357_b200/variants/libmobile_nohold.so python scripts/ab_dp.py c2 nohold
python scripts/trace_dp.py c3 little > gpurun_out/r2_trace_hold.json
python -c "import json;d=json.load(open('gpurun_out/r2_trace_hold.json'));print(json.dumps(d['per_kind']))"
