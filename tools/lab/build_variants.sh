#!/bin/bash
# Builds A/B variants of liblatsum_cuda.so from expand.cu with extra -D flags (development only:
# experimental #ifdef blocks are added to the kernel temporarily) into
# lab_build/<name>/paper_1405_2270_b200/. Usage: build_variants.sh name:"-DX -DY" ...
set -e
ROOT=/root/repo
PKG=$ROOT/paper_1405_2270_b200
ARCH="-gencode arch=compute_100a,code=sm_100a"
SRC=${SRC:-expand}  # which csrc/<SRC>.cu the flags apply to
OTHERS=$(ls $ROOT/build/obj/*.o | grep -v "/$SRC.o$")
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  d=$ROOT/${LAB_DIR:-lab_build}/$name/paper_1405_2270_b200
  mkdir -p $d
  cp $PKG/*.py $d/
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$ROOT/include $flags -c $PKG/csrc/$SRC.cu -o $d/$SRC.o &
done
wait
for spec in "$@"; do
  name=${spec%%:*}
  d=$ROOT/${LAB_DIR:-lab_build}/$name/paper_1405_2270_b200
  nvcc $ARCH -shared -o $d/liblatsum_cuda.so $d/$SRC.o $OTHERS -lcudart
  rm $d/$SRC.o
done
