O=gpurun_out/$1; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fate_score -s 3 -c 1 -o $O/c5_full python bench.py --steps 3 --warmup 3 --no-cpu --no-c4 --no-c2 > $O/ncu_c5.log 2>&1
