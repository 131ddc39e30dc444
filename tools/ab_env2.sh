#!/bin/bash
# A/B of environment settings on an A/B library build (FATE_BUILD_AB=1):
# tools/ab_env2.sh OUTDIR LIB "NAME=VAL ..." ...
O=$1; shift
L=$1; shift
mkdir -p $O
cp paper_2605_07238_b200/libfate.so /tmp/libfate_orig.so
cp $L paper_2605_07238_b200/libfate.so
for pass in 1 2; do
  for cfg in "$@"; do
    env $cfg KB_TAG="$cfg-$pass" timeout 600 python tools/kbench.py 30 3 >> $O/kbench.jsonl 2>> $O/kbench.err
  done
done
cp /tmp/libfate_orig.so paper_2605_07238_b200/libfate.so
