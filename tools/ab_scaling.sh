#!/bin/bash
# A/B of library variants on the strong-scaling shards (tools/shard_scaling.py):
# tools/ab_scaling.sh OUTDIR "ARGS" lib1.so lib2.so ...
O=$1; shift
A=$1; shift
mkdir -p $O
cp paper_2605_07238_b200/libfate.so /tmp/libfate_orig.so
for pass in 1 2; do
  for l in "$@"; do
    cp $l paper_2605_07238_b200/libfate.so
    echo "{\"lib\": \"$(basename $l)-$pass\"}" >> $O/scal.jsonl
    timeout 900 python tools/shard_scaling.py $A >> $O/scal.jsonl 2>> $O/scal.err
  done
done
cp /tmp/libfate_orig.so paper_2605_07238_b200/libfate.so
