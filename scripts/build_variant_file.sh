#!/bin/bash
# build_variant_file.sh SRC NAME "NVCC FLAGS": libdso_b200_NAME.so with SRC.cu compiled with
# extra flags (experiment builds for scripts/variants.sh; not used by tests or the bench)
set -e
cd "$(dirname "$0")/../paper_2407_13096_b200/csrc"
SRC=$1; NAME=$2; FLAGS=$3
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $FLAGS -c $SRC.cu -o build/${SRC}_v_$NAME.o
OBJS=$(ls build/*.o | grep -v "/${SRC}\.o\|_v_\|mlp_phase\|mlp_nosweep\|mlp_noprod\|tcprobe")
nvcc $ARCH -shared -o ../lib/libdso_b200_$NAME.so $OBJS build/${SRC}_v_$NAME.o -lcudart -ldl
echo built ../lib/libdso_b200_$NAME.so
