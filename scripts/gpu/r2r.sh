python scripts/ab_dp.py c3 base
MOBILE_LIB=paper_2510_12357_b200/variants/libmobile_nofma.so python scripts/ab_dp.py c3 nofma
python scripts/ab_dp.py c2 base
MOBILE_LIB=paper_2510_12357_b200/variants/libmobile_nofma.so python scripts/ab_dp.py c2 nofma
