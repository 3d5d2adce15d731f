OUT=${OUT:-r3d}; mkdir -p gpurun_out/$OUT
timeout 900 python -m pytest tests/test_sparse_gpu.py -q -x > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
timeout 600 python tools/c3_sparse.py 128 64 148 3 > gpurun_out/$OUT/c3m_sparse.txt 2>&1
timeout 900 python tools/c3_sparse.py 256 180 148 1 > gpurun_out/$OUT/c3full_sparse_148.txt 2>&1
