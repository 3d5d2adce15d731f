#!/bin/bash
# select_screen: warp sorts + merge
OUT=${OUT:-r6h}; mkdir -p gpurun_out/$OUT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -2 gpurun_out/$OUT/pytest.log
timeout 900 python tools/c3_sparse.py 256 180 148 1 20 > gpurun_out/$OUT/c3full_148x1.txt 2>&1
timeout 600 python tools/c3_sparse.py 128 64 148 3 100 > gpurun_out/$OUT/c3m_148x3.txt 2>&1
python tools/prof_c5.py 296 20 > gpurun_out/$OUT/c5.txt 2>&1
python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps.txt 2>&1
cat gpurun_out/$OUT/c3*.txt gpurun_out/$OUT/c5.txt
python -c "
import json
for l in open('gpurun_out/$OUT/ps.txt'):
    if l.startswith('{'): d=json.loads(l); print(d['config'], d['us_per_iteration'], d['best']==d['golden_best'])"
