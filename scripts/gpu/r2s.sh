python scripts/ab_dp.py c3 base
for kb in 64 128 256 512 1024; do MOBILE_DP_PF_KB=$kb python scripts/ab_dp.py c3 pf$kb; done
for kb in 128 512; do MOBILE_DP_PF_KB=$kb python scripts/ab_dp.py c2 pf$kb; done
python scripts/ab_dp.py c2 base
