#!/bin/bash
OUT=${OUT:-r6g}; mkdir -p gpurun_out/$OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve --launch-count 1 \
    -o gpurun_out/$OUT/c3full -f python tools/c3_sparse.py 256 180 1 1 20 > gpurun_out/$OUT/ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/$OUT/ncu.log
