#!/bin/bash
# A/B bench over environment settings: tools/ab_env.sh OUTDIR "NAME=VAL ..." ...
O=$1; shift
mkdir -p $O
k=0
for cfg in "$@"; do
  k=$((k+1))
  env $cfg timeout 300 python bench.py --no-cpu --steps 30 > $O/bench_$k.json 2> $O/bench_$k.err
  echo "$k: $cfg" >> $O/configs.txt
done
