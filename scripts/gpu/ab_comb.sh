for c in c3 c2 c4; do
python scripts/ab_perop.py $c sep
MOBILE_FUSE_COMBINE=1 python scripts/ab_perop.py $c fused
done
MOBILE_FUSE_COMBINE=1 timeout 900 python -m pytest tests/test_runtime_gpu.py tests/test_decode_gpu.py tests/test_functional_gpu.py -x -q 2>&1 | tail -2
