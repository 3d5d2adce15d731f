#!/bin/bash
OUT=${OUT:-r5h}; mkdir -p gpurun_out/$OUT
timeout 600 python tools/c3_sparse.py 256 180 3 1 20 > gpurun_out/$OUT/c3full_3x1.txt 2>&1
timeout 600 python tools/c3_sparse.py 256 180 1 2 20 > gpurun_out/$OUT/c3full_1x2.txt 2>&1
cat gpurun_out/$OUT/*.txt
