#!/bin/bash
# full suite + default bench (all legs incl. the full-size C3 leg)
OUT=${OUT:-r6a}; mkdir -p gpurun_out/$OUT
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -2 gpurun_out/$OUT/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$OUT/smoke.log 2>&1; tail -1 gpurun_out/$OUT/smoke.log
SECONDS=0; timeout 1800 python bench.py > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err; echo "bench rc=$?"
echo "bench seconds $SECONDS"
python -c "
import json; d=json.loads(open('gpurun_out/$OUT/bench.json').read().strip().split(chr(10))[-1])
print(d['value'], d['parity']['bitwise'], d['roofline']['frac'], [(t['config'], t['gpu_wall_s'], t['cpu_port_wall_s'], t['gpu_vs_cpu_port']) for t in d['time_to_reference_linf']])
w=d['workloads']; print({k:(v['value'], v['parity']) for k,v in w.items()}); print(w['c3_slices'].get('dense_engine'))"
