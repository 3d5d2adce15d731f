OUT=${OUT:-r2t}; mkdir -p gpurun_out/$OUT
timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_gpu_parity.py -q -x > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-ttr > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err; echo "bench rc=$?" >> gpurun_out/$OUT/bench.err
