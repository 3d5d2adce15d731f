#!/bin/bash
OUT=${OUT:-r4i}; mkdir -p gpurun_out/$OUT
for c in c2 c1; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve --launch-skip 1 --launch-count 1 \
    -o gpurun_out/$OUT/$c -f python tools/solve_one.py $c > gpurun_out/$OUT/ncu_$c.log 2>&1
done
