#!/bin/bash
# One GPU session: parity tests, smoke, bench (both arms).
# usage: tools/gpu_session.sh TAG [pytest -k expr]
O=gpurun_out/$1
mkdir -p $O
ls baseline/_ref > $O/ref_ls.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
K=${2:+-k "$2"}
timeout 1800 python -m pytest tests -m gpu -x -q $K --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
ls -la $O
