#!/bin/bash
# Builds a lab variant of liblatsum_cuda.so with extra -D flags (e.g. "-DLS_DEV_KNOBS
# -DLS_TIMELINE") into lab_build/<name>/paper_1405_2270_b200/ (git- and gpurun-ignored? no:
# lab_build/ is gpurun-ignored, so copy the result next to the repo for a GPU run with
# LS_LAB_ROOT). Usage: build_lab.sh name "FLAGS"
set -e
ROOT=/root/repo
PKG=$ROOT/paper_1405_2270_b200
ARCH="-gencode arch=compute_100a,code=sm_100a"
name=$1; flags=$2
d=$ROOT/${LAB_DIR:-lab_build}/$name/paper_1405_2270_b200
mkdir -p $d/obj
cp $PKG/*.py $d/
for src in $PKG/csrc/*.cu; do
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$ROOT/include $flags -c $src -o $d/obj/$(basename $src .cu).o &
done
wait
nvcc $ARCH -shared -o $d/liblatsum_cuda.so $d/obj/*.o -lcudart
rm -rf $d/obj
echo $d/liblatsum_cuda.so
