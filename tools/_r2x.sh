OUT=${OUT:-r2x}; mkdir -p gpurun_out/$OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_api_gpu.py tests/test_layer_gpu.py -q -x > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps.txt 2>&1
FCPROF=1 AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_fcprof.so python tools/phase_single.py c1 c2 > gpurun_out/$OUT/fcprof.txt 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-ttr --no-e2e --no-legs > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err
