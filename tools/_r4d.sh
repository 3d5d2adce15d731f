#!/bin/bash
# ncu source-level stall profile of the single-instance solves (C1, C2)
OUT=${OUT:-r4d}; mkdir -p gpurun_out/$OUT
python tools/solve_one.py c2 && python tools/solve_one.py c1
for c in c2 c1; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve --launch-skip 1 --launch-count 1 \
    -o gpurun_out/$OUT/$c -f python tools/solve_one.py $c > gpurun_out/$OUT/ncu_$c.log 2>&1
  echo "$c ncu rc=$?"
done
