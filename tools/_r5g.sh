#!/bin/bash
OUT=${OUT:-r5g}; mkdir -p gpurun_out/$OUT
FCPROF=1 AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_fcprof.so python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps_fcprof.txt 2>&1
timeout 1800 python bench.py > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err; echo "bench rc=$?"
cat gpurun_out/$OUT/ps_fcprof.txt
python -c "
import json; d=json.loads(open('gpurun_out/$OUT/bench.json').read().strip().split(chr(10))[-1])
print(d['value'], d['parity']['bitwise'], d['roofline']['frac'], [(t['config'], t['gpu_wall_s'], t['cpu_port_wall_s'], t['gpu_vs_cpu_port']) for t in d['time_to_reference_linf']])
w=d['workloads']; print({k:(v['value'], v['parity']) for k,v in w.items()}); print(w['c3_full'])"
tail -5 gpurun_out/$OUT/bench.err
