set -x
OUT=r2a; mkdir -p gpurun_out/$OUT
( lscpu | head -20; nproc; python -c "import numpy; from threadpoolctl import threadpool_info; print(threadpool_info())" ) > gpurun_out/$OUT/host.txt 2>&1
timeout 900 python -m pytest tests/test_api_gpu.py tests/test_layer_gpu.py -x -q > gpurun_out/$OUT/pytest_new.log 2>&1; echo "pytest_new rc=$?" >> gpurun_out/$OUT/pytest_new.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err; echo "bench rc=$?"
