#!/bin/bash
# The bench's multi-rank plan end to end on ONE GPU (validation only):
# 2 and 4 ranks over gloo, every rank on cuda:0.  Checks gather_check / host
# solve / weak / c4 split plumbing; the timings are not scaling numbers.
O=gpurun_out/$1
mkdir -p $O
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 5 \
    --warmup 3 --dist-backend gloo --share-device --no-cpu --no-c2 > $O/bench_n$n.json 2> $O/bench_n$n.err
  echo "n=$n rc=$?" >> $O/rc.txt
done
