OUT=${OUT:-r3c}; mkdir -p gpurun_out/$OUT
timeout 900 python -m pytest tests/test_sparse_gpu.py -q -x > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_fcprof.so timeout 600 python tools/c3_sparse.py 128 64 148 2 > gpurun_out/$OUT/c3m_sparse_fcprof.txt 2>&1
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_fcprof.so timeout 600 python tools/c3_sparse.py 128 64 148 2 100 --dense > gpurun_out/$OUT/c3m_dense_fcprof.txt 2>&1
