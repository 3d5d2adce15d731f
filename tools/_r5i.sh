#!/bin/bash
OUT=${OUT:-r5i}; mkdir -p gpurun_out/$OUT
timeout 600 python tools/c3_sparse.py 256 180 3 1 20 > gpurun_out/$OUT/c3full_3x1.txt 2>&1
timeout 900 python -m pytest tests/test_sparse_gpu.py tests/test_c3full_gpu.py -x -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
timeout 600 python tools/c3_sparse.py 256 180 148 1 20 > gpurun_out/$OUT/c3full_148x1.txt 2>&1
tail -2 gpurun_out/$OUT/pytest.log
cat gpurun_out/$OUT/c3full*.txt
