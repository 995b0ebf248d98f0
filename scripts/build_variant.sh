#!/bin/bash
# build_variant.sh NAME "NVCC FLAGS": libdso_b200_NAME.so with mlp.cu compiled with extra
# flags (experiment builds for scripts/variants.sh; not used by tests or the bench)
set -e
cd "$(dirname "$0")/../paper_2407_13096_b200/csrc"
NAME=$1; FLAGS=$2
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $FLAGS -c mlp.cu -o build/mlp_v_$NAME.o
OBJS=$(ls build/*.o | grep -v "mlp\.o\|mlp_phase\|mlp_nosweep\|mlp_noprod\|mlp_v_\|tcprobe")
nvcc $ARCH -shared -o ../lib/libdso_b200_$NAME.so $OBJS build/mlp_v_$NAME.o -lcudart -ldl
echo built ../lib/libdso_b200_$NAME.so
