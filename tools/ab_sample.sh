#!/bin/bash
# A/B of sampler builds on one launch (dev tooling).  Variants are in-tree builds of the
# library, e.g.  make -C paper_2208_00613_b200/csrc XDEFS="-DIMMX_BLK_U=5" OUT=../../variants/var_u5.so BUILD=../../build/obj_u5
# usage: tools/ab_sample.sh <config> <samples> main|<name>...   (<name> -> variants/var_<name>.so)
cfg=$1; cnt=$2; shift 2
for r in 1 2; do
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib=$PWD/variants/var_$v.so; fi
  echo "== $v"; IMMX_B200_LIB=$lib timeout 300 python tools/prof_sample.py --config $cfg --count $cnt --reps 2 2>&1 | grep "rep 1"
done; done
