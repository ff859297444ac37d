#!/bin/bash
# build_any.sh NAME FILE.cu "-DDEFINES..." : variant build of one source file -> _lib/libtmfg_b200_NAME.so
set -e
D=$(cd "$(dirname "$0")/../paper_2408_09399_b200/csrc" && pwd)
L=$D/../_lib
F=$2
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -DTM_PROFILE=0 $3 \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -ccbin /usr/bin/g++ -c $D/$F -o /tmp/${F%.cu}_$1.o
objs=$(ls $L/obj/*.o | grep -v "/${F%.cu}.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -fPIC $objs /tmp/${F%.cu}_$1.o -o $L/libtmfg_b200_$1.so
echo built $L/libtmfg_b200_$1.so
