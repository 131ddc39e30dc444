#!/bin/bash
# drop-in path check: GPU golden/compat/mirror tests + the c2_fate_runs and api_build_problem timings
O=gpurun_out/$1; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -k "golden or compat or mirror" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python -c "
import json, bench
print(json.dumps({'c2': bench.measure_c2_runs(), 'api': bench.measure_api_waves()}))" > $O/c2.json 2> $O/c2.err
