#!/bin/bash
# swap-eval pruning, narrow impact tile, radix compaction, pairs threshold 4
OUT=${OUT:-r4c}; mkdir -p gpurun_out/$OUT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -2 gpurun_out/$OUT/pytest.log
python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps.txt 2>&1
FCPROF=1 AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_fcprof.so python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps_fcprof.txt 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-legs > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err
cat gpurun_out/$OUT/ps*.txt
