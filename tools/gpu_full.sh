#!/bin/bash
# One full GPU session: GPU test suite, smoke, bench (both arms), ncu launch
# list of the bench command, one ncu --set full capture per workload.
# usage: tools/gpu_full.sh TAG
set -x
O=gpurun_out/$1
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=20 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-c4 --no-c2 > $O/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fate_score -s 3 -c 1 -o $O/c5_full python bench.py --steps 3 --warmup 3 --no-cpu --no-c4 --no-c2 > $O/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fate_score -s 3 -c 1 -o $O/c4_full python bench.py --workload c4 --mode sweep --steps 3 --warmup 3 --no-cpu --no-c2 > $O/ncu_c4.log 2>&1
ls -la $O
