#!/bin/bash
# usage: variant.sh NAME "-DFLAGS"  -> paper_2405_04416_b200/libdg_NAME.so (kernels_mlp_tc.cu recompiled)
set -e
cd /root/repo
NAME=$1; shift
OBJ=build/obj
mkdir -p build/var
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3 -Iinclude -Ipaper_2405_04416_b200/csrc --expt-relaxed-constexpr "$@" -c paper_2405_04416_b200/csrc/kernels_mlp_tc.cu -o build/var/mlp_tc_$NAME.o
objs=$(ls $OBJ/*.o | grep -v kernels_mlp_tc.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2405_04416_b200/libdg_$NAME.so $objs build/var/mlp_tc_$NAME.o -ldl -lpthread
