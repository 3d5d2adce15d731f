#!/bin/bash
OUT=${OUT:-r4k}; mkdir -p gpurun_out/$OUT
python tools/prof_c5.py 296 20 > gpurun_out/$OUT/plain.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve --launch-count 1 \
    -o gpurun_out/$OUT/c5 -f python tools/prof_c5.py 296 20 > gpurun_out/$OUT/ncu_c5.log 2>&1
cat gpurun_out/$OUT/plain.txt
