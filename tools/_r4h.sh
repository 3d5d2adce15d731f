#!/bin/bash
# division-free filter bound test
OUT=${OUT:-r4h}; mkdir -p gpurun_out/$OUT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -2 gpurun_out/$OUT/pytest.log
python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps.txt 2>&1
cat gpurun_out/$OUT/ps*.txt
