#!/bin/bash
# A/B of library variants on the drop-in path timing (bench.measure_c2_runs):
# tools/ab_c2.sh OUTDIR lib1.so lib2.so ...
O=$1; shift
mkdir -p $O
cp paper_2605_07238_b200/libfate.so /tmp/libfate_orig.so
for pass in 1 2; do
  for l in "$@"; do
    cp $l paper_2605_07238_b200/libfate.so
    timeout 900 python -c "
import json, bench
r = bench.measure_c2_runs()
print(json.dumps({'lib': '$(basename $l)-$pass', 'gpu_policy_s': r['gpu_policy_s'], 'per_wave_ms': r['gpu_score_ms_per_wave_excl_bank_setup'], 'mirror_s': r['gpu_mirror_durations_s'], 'ref_s': r['reference_python_s']}))" >> $O/c2.jsonl 2>> $O/c2.err
  done
done
cp /tmp/libfate_orig.so paper_2605_07238_b200/libfate.so
