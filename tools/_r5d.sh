#!/bin/bash
# final bench line + launch list + workspace sizes
OUT=${OUT:-r5d}; mkdir -p gpurun_out/$OUT
timeout 1500 python bench.py > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/$OUT/bench_ref.json 2> gpurun_out/$OUT/bench_ref.err; echo "ref rc=$?"
python tools/ws_sizes.py > gpurun_out/$OUT/ws.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-ttr --no-legs > gpurun_out/$OUT/ncu_bench.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/$OUT/ws.txt
tail -c 600 gpurun_out/$OUT/bench_ref.json
python -c "import json; d=json.loads(open('gpurun_out/$OUT/bench.json').read().strip().split(chr(10))[-1]); print(d['value'], d['e2e']['value'], d['parity']['bitwise'], d['roofline']['frac'], d['clocks'], [(t['config'], t['gpu_vs_cpu_port']) for t in d['time_to_reference_linf']])"
