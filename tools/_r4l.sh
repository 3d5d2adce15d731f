#!/bin/bash
# dual CTA size (512 x 1 for count <= SMs)
OUT=${OUT:-r4l}; mkdir -p gpurun_out/$OUT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -2 gpurun_out/$OUT/pytest.log
python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps.txt 2>&1
python tools/prof_c5.py 296 20 > gpurun_out/$OUT/c5.txt 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-legs > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err
cat gpurun_out/$OUT/ps.txt gpurun_out/$OUT/c5.txt
python -c "import json; d=json.loads(open('gpurun_out/$OUT/bench.json').read().strip().split(chr(10))[-1]); print(d['value'], d['parity']['bitwise'], d['k_solve']['phase_share'], [(t['config'], t['gpu_vs_cpu_port']) for t in d['time_to_reference_linf']])"
