#!/bin/bash
OUT=${OUT:-r6i}; mkdir -p gpurun_out/$OUT
timeout 900 python -m pytest tests/test_layer_gpu.py -x -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -2 gpurun_out/$OUT/pytest.log
for k in 1 2; do
python tools/prof_c5.py 296 20 > gpurun_out/$OUT/c5_base$k.txt 2>&1
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_ic8.so python tools/prof_c5.py 296 20 > gpurun_out/$OUT/c5_ic8$k.txt 2>&1
done
head -1 gpurun_out/$OUT/c5_*.txt
