#!/bin/bash
# 512-thread engine (diag build): parity + single-instance latency + C5 throughput
OUT=${OUT:-r5e}; mkdir -p gpurun_out/$OUT
L=$PWD/paper_2508_13437_b200/libamvm_nt512.so
AMVM_LIBRARY=$L timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_layer_gpu.py tests/test_sparse_gpu.py tests/test_api_gpu.py -x -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -3 gpurun_out/$OUT/pytest.log
AMVM_LIBRARY=$L python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps512.txt 2>&1
python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps256.txt 2>&1
AMVM_LIBRARY=$L python tools/prof_c5.py 296 20 > gpurun_out/$OUT/c5_512.txt 2>&1
python tools/prof_c5.py 296 20 > gpurun_out/$OUT/c5_256.txt 2>&1
for f in ps512 ps256; do python -c "
import json,sys
for l in open('gpurun_out/$OUT/$f.txt'):
    if l.startswith('{'): d=json.loads(l); print('$f', d['config'], d['us_per_iteration'], d['best']==d['golden_best'])
"; done
head -2 gpurun_out/$OUT/c5_512.txt gpurun_out/$OUT/c5_256.txt
