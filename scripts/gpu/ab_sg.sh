# A/B of the streaming GEMV ring geometry (variants built by scripts/build_variant.sh with SRC=stream_gemv.cu)
mkdir -p gpurun_out
for lib in ${LIBS:-default sg3k4 sg2k5}; do
  if [ $lib = default ]; then L=paper_2510_12357_b200/libmobile.so; else L=paper_2510_12357_b200/variants/libmobile_$lib.so; fi
  for m in c5 c2 c3; do MOBILE_LIB=$L timeout 300 python scripts/ab_perop.py $m $lib 2>&1 | tail -1; done
done > gpurun_out/r2_ab_sg.txt
cat gpurun_out/r2_ab_sg.txt
for lib in ${TLIBS:-sg3k4 sg2k5}; do
  MOBILE_LIB=paper_2510_12357_b200/variants/libmobile_$lib.so timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_runtime_gpu.py -q -x -k "gemv or head or step_engine or moe_layer or attn" 2>&1 | tail -2
done
