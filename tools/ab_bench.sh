#!/bin/bash
# A/B kernel-only timing of scoring kernel generations on C5 frontier and C4 sweep.
# usage: tools/ab_bench.sh OUTDIR gen1 gen2 ...
O=$1; shift
mkdir -p $O
for g in "$@"; do
  FATE_SCORE_KERNEL=$g timeout 300 python bench.py --no-cpu --steps 30 > $O/bench_$g.json 2> $O/bench_$g.err
done
