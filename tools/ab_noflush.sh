#!/bin/bash
# warm-L2 upper bound: the production library timed with and without the L2 flush
O=gpurun_out/$1; mkdir -p $O
for pass in 1 2; do
  KB_TAG=flush-$pass timeout 600 python tools/kbench.py 30 3 >> $O/kbench.jsonl 2>> $O/kbench.err
  KB_TAG=noflush-$pass KB_NOFLUSH=1 timeout 600 python tools/kbench.py 30 3 >> $O/kbench.jsonl 2>> $O/kbench.err
done
