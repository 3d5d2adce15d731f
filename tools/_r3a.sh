OUT=${OUT:-r3a}; mkdir -p gpurun_out/$OUT
timeout 600 python tools/c3_sparse.py 128 64 148 3 > gpurun_out/$OUT/c3m_sparse.txt 2>&1
timeout 600 python tools/c3_sparse.py 128 64 148 3 100 --dense > gpurun_out/$OUT/c3m_dense.txt 2>&1
timeout 900 python tools/c3_sparse.py 256 180 16 1 > gpurun_out/$OUT/c3full_sparse_16.txt 2>&1
timeout 900 python tools/c3_sparse.py 256 180 148 1 > gpurun_out/$OUT/c3full_sparse_148.txt 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-ttr --no-e2e --no-legs > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err
