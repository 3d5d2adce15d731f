OUT=${OUT:-r2y}; mkdir -p gpurun_out/$OUT
timeout 900 python bench.py --steps 2 --warmup 3 --no-ttr --no-e2e --no-legs > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err; echo "bench rc=$?" >> gpurun_out/$OUT/bench.err
