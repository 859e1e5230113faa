#!/bin/bash
# Build paper_2510_12357_b200/variants/libmobile_<name>.so: the in-tree objects
# with decode_pass.cu (or SRC=<file>.cu) recompiled under extra -D flags (A/B experiments on the
# box: MOBILE_LIB=... python scripts/trace_dp.py).
#   scripts/build_variant.sh <name> [-DFOO=1 ...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
src=${SRC:-decode_pass.cu}
mkdir -p paper_2510_12357_b200/variants /tmp/variant_$name
python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2510_12357_b200/build.py'); m=u.module_from_spec(s); s.loader.exec_module(m); m.build()"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O3 -I include \
  --expt-relaxed-constexpr -Xptxas -O3 "$@" -c paper_2510_12357_b200/csrc/$src -o /tmp/variant_$name/${src%.cu}.o
objs=$(ls paper_2510_12357_b200/build/*.o | grep -v $src.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2510_12357_b200/variants/libmobile_$name.so $objs /tmp/variant_$name/${src%.cu}.o
echo paper_2510_12357_b200/variants/libmobile_$name.so
