#!/bin/bash
# sparse one_opt: argmax-row column screen
OUT=${OUT:-r5j}; mkdir -p gpurun_out/$OUT
timeout 900 python -m pytest tests/test_sparse_gpu.py tests/test_c3full_gpu.py -x -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -3 gpurun_out/$OUT/pytest.log
timeout 600 python tools/c3_sparse.py 256 180 3 1 20 > gpurun_out/$OUT/c3full_3x1.txt 2>&1
timeout 900 python tools/c3_sparse.py 256 180 148 1 20 > gpurun_out/$OUT/c3full_148x1.txt 2>&1
timeout 600 python tools/c3_sparse.py 128 64 148 3 100 > gpurun_out/$OUT/c3m_148x3.txt 2>&1
cat gpurun_out/$OUT/c3*.txt
