#!/bin/bash
# A/B kernel timing of prebuilt library variants: tools/ab_libs.sh OUTDIR lib1.so lib2.so ...
# Each variant is copied over paper_2605_07238_b200/libfate.so and timed by
# tools/kbench.py (twice, interleaved, to expose box drift).
O=$1; shift
mkdir -p $O
cp paper_2605_07238_b200/libfate.so /tmp/libfate_orig.so
for pass in 1 2; do
  for l in "$@"; do
    cp $l paper_2605_07238_b200/libfate.so
    KB_TAG=$(basename $l)-$pass timeout 600 python tools/kbench.py 30 3 >> $O/kbench.jsonl 2>> $O/kbench.err
  done
done
cp /tmp/libfate_orig.so paper_2605_07238_b200/libfate.so
