#!/bin/bash
# violation-row screen for swaps, radix early exit, warp bucket sort
OUT=${OUT:-r4f}; mkdir -p gpurun_out/$OUT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -2 gpurun_out/$OUT/pytest.log
python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps.txt 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-legs > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err
for c in c1 c2; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve --launch-skip 1 --launch-count 1 \
    -o gpurun_out/$OUT/$c -f python tools/solve_one.py $c > gpurun_out/$OUT/ncu_$c.log 2>&1
done
cat gpurun_out/$OUT/ps*.txt
python -c "import json; d=json.loads(open('gpurun_out/$OUT/bench.json').read().strip().split(chr(10))[-1]); print(d['value'], d['parity']['bitwise'], [(t['config'], t['gpu_vs_cpu_port']) for t in d['time_to_reference_linf']])"
