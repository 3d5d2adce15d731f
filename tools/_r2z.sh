OUT=${OUT:-r2z}; mkdir -p gpurun_out/$OUT
timeout 900 python -m pytest tests/test_sparse_gpu.py -q -x > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_api_gpu.py -q -x > gpurun_out/$OUT/pytest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest2.log
