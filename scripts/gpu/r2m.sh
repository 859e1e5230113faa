for nc in 9 4 2 1; do
MOBILE_DP_ATTN_NC=$nc python scripts/ab_dp.py c3 nc$nc
MOBILE_DP_ATTN_NC=$nc python scripts/ab_dp.py c2 nc$nc
done
for nc in 4 2 1; do MOBILE_DP_ATTN_NC=$nc python scripts/ab_dp.py c5 nc$nc; done
MOBILE_DP_ATTN_NC=1 timeout 600 python -m pytest tests/test_decode_pass_gpu.py -x -q 2>&1 | tail -2
