#!/bin/bash
O=$1; shift
mkdir -p $O
for i in "$@"; do
  FATE_V6_IPC=$i timeout 300 python bench.py --no-cpu --steps 30 > $O/bench_ipc$i.json 2> $O/bench_ipc$i.err
done
