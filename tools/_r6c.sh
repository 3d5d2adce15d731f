#!/bin/bash
OUT=${OUT:-r6c}; mkdir -p gpurun_out/$OUT
timeout 2400 python -m pytest tests -m gpu -q --durations=6 > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -12 gpurun_out/$OUT/pytest.log
