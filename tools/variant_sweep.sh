#!/bin/bash
# Time every variants/libswedg_<name>.so given on the command line with tools/kprobe.py.
#   tools/variant_sweep.sh "MODAL_K1D SBP_K1D STEPS" name1 name2 ...
args=$1; shift
for v in "$@"; do
  echo "== $v"
  SWEDG_LIB_VARIANT=variants/libswedg_$v.so python tools/kprobe.py $args 2>&1 | grep -v "fp64 peak"
done
