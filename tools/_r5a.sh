#!/bin/bash
# round-2 evidence: full GPU suite (incl. the full-size C3 oracle golden), smoke, default bench
OUT=${OUT:-r5a}; mkdir -p gpurun_out/$OUT
timeout 2400 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -14 gpurun_out/$OUT/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$OUT/smoke.log 2>&1; tail -1 gpurun_out/$OUT/smoke.log
timeout 1500 python bench.py > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/$OUT/bench.json').read().strip().split(chr(10))[-1]); print(d['value'], d['parity']['bitwise'], d['roofline']['frac'], d['roofline'].get('without_pdl'), [(t['config'], t['gpu_vs_cpu_port']) for t in d['time_to_reference_linf']])"
