#!/bin/bash
# Build an alternative libswedg_b200.so with extra nvcc flags (e.g. -DSWEDG_PAIR_LB2=0)
# into variants/libswedg_<name>.so; select it at run time with SWEDG_LIB_VARIANT=<path>.
#   tools/build_variant.sh NAME [nvcc flags...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off -shared -Xptxas -v "$@" \
  paper_2005_02516_b200/csrc/swedg_capi.cu paper_2005_02516_b200/csrc/setup.cpp \
  -o variants/libswedg_$name.so 2> variants/ptxas_$name.txt
grep -A3 "modal_volume_pair_n4_kernelILb0" variants/ptxas_$name.txt | grep -E "spill|registers" | tr '\n' ' '; echo " [$name]"
