#!/bin/bash
# A/B of environment settings of an A/B library build on the strong-scaling
# shards: tools/ab_scaling_env.sh OUTDIR LIB "NAME=VAL ..." ...
O=$1; shift
L=$1; shift
mkdir -p $O
cp paper_2605_07238_b200/libfate.so /tmp/libfate_orig.so
cp $L paper_2605_07238_b200/libfate.so
for cfg in "$@"; do
  echo "{\"lib\": \"$cfg\"}" >> $O/scal.jsonl
  env $cfg timeout 600 python tools/shard_scaling.py 30 >> $O/scal.jsonl 2>> $O/scal.err
done
cp /tmp/libfate_orig.so paper_2605_07238_b200/libfate.so
