#!/bin/bash
# build_variant.sh NAME [ENV=VAL ...]: copy csrc to /tmp, regenerate the solve with the
# given generator settings, build tools/libsvk_NAME.so (for SVK_LIBRARY A/B runs).
set -e
NAME=$1; shift
D=/tmp/svkvar_$NAME/pkg; rm -rf /tmp/svkvar_$NAME; mkdir -p $D /tmp/svkvar_$NAME/include; cp include/*.h /tmp/svkvar_$NAME/include/
cp -r paper_2401_06277_b200/csrc $D/
env "$@" python tools/gen_solve.py $D/csrc > /dev/null
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -shared -Xcompiler -fPIC -lineinfo -gencode arch=compute_100a,code=sm_100a \
  -Xptxas -v --expt-relaxed-constexpr $NVFLAGS -Iinclude $D/csrc/svk.cu -o tools/libsvk_$NAME.so > $D/build.log 2>&1
python tools/ptxas_summary.py $D/build.log | grep vanka
