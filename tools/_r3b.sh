OUT=${OUT:-r3b}; mkdir -p gpurun_out/$OUT
timeout 900 python -m pytest tests/test_sparse_gpu.py tests/test_gpu_parity.py tests/test_tomo_gpu.py -q -x > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-ttr --no-e2e --no-legs > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err
timeout 600 python tools/c3_sparse.py 128 64 148 3 > gpurun_out/$OUT/c3m_sparse.txt 2>&1
timeout 900 python tools/c3_sparse.py 256 180 148 1 > gpurun_out/$OUT/c3full_sparse_148.txt 2>&1
