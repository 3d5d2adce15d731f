OUT=${OUT:-r2v}; mkdir -p gpurun_out/$OUT
timeout 600 python -m pytest tests/test_tomo_gpu.py tests/test_api_gpu.py -q -x > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
timeout 1200 python bench.py --steps 2 --warmup 3 > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err; echo "bench rc=$?" >> gpurun_out/$OUT/bench.err
