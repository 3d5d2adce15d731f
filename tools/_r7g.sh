#!/bin/bash
OUT=${OUT:-r7g}; mkdir -p gpurun_out/$OUT
for k in 1 2; do
python tools/prof_c5.py 296 20 > gpurun_out/$OUT/c5_base$k.txt 2>&1
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_rp12.so python tools/prof_c5.py 296 20 > gpurun_out/$OUT/c5_rp12$k.txt 2>&1
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_ds32.so python tools/prof_c5.py 296 20 > gpurun_out/$OUT/c5_ds32$k.txt 2>&1
done
for f in gpurun_out/$OUT/c5_*.txt; do echo $f; head -1 $f | grep -o "'find_cand': np.float64([0-9.]*)"; done
