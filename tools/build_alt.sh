#!/bin/bash
# Dev aid: lib/libeh_alt.so = the current objects with ONE source recompiled under extra
# flags (A/B runs inside one gpurun call: TRI_LIB=paper_1503_02368_b200/lib/libeh_alt.so).
#   tools/build_alt.sh count_tri.cu -DEH_HASH_FILTER=0
set -e
P=paper_1503_02368_b200; SRC=$1; shift
python -c "from paper_1503_02368_b200 import build; build.build()"
O=/tmp/alt_${SRC%.cu}.o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O3 \
  --expt-relaxed-constexpr -Xptxas -warn-spills "$@" -I include -I $P/csrc -c $P/csrc/$SRC -o $O
OBJS=$(ls $P/lib/obj/*.o | grep -v "/${SRC%.cu}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/lib/libeh_alt.so $OBJS $O -lcudart
echo built $P/lib/libeh_alt.so
