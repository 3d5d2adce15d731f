#!/bin/bash
OUT=${OUT:-r4g}; mkdir -p gpurun_out/$OUT
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/$OUT/mem.txt
timeout 1500 python -m pytest tests/test_c3full_gpu.py -x -q --durations=5 > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -15 gpurun_out/$OUT/pytest.log
