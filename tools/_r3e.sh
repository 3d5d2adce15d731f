OUT=${OUT:-r3e}; mkdir -p gpurun_out/$OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_layer_gpu.py tests/test_sparse_gpu.py -q -x > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-ttr --no-e2e --no-legs > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err
python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps.txt 2>&1
