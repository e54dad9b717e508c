#!/bin/bash
# build a variant of libvoxschur.so with extra -D flags for vs_cgx.cu (same-box A/B experiments):
#   tools/build_variant.sh NAME -DVS_X_FMA=7 ...   ->  _ab/lib_NAME.so   (use with VOXSCHUR_LIB)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2307_05266_b200/csrc"
mkdir -p ../../_ab
nvcc -O3 -lineinfo -fmad=false -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O2 -gencode arch=compute_100a,code=sm_100a "$@" -c vs_cgx.cu -o /tmp/vs_cgx_$name.o
objs=$(ls _obj/*.o | grep -v vs_cgx.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static $objs /tmp/vs_cgx_$name.o -o ../../_ab/lib_$name.so
