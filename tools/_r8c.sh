#!/bin/bash
OUT=${OUT:-r8c}; mkdir -p gpurun_out/$OUT
for k in 1 2; do
python tools/phase_single.py c1 > gpurun_out/$OUT/base$k.txt 2>&1
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_pm8.so python tools/phase_single.py c1 > gpurun_out/$OUT/pm8$k.txt 2>&1
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_pm2.so python tools/phase_single.py c1 > gpurun_out/$OUT/pm2$k.txt 2>&1
done
for f in gpurun_out/$OUT/*.txt; do python -c "
import json
for l in open('$f'):
    if l.startswith('{'): d=json.loads(l); print('$f', d['config'], d['us_per_iteration'], d['best']==d['golden_best'])"; done
