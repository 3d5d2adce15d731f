OUT=${OUT:-r2s}; mkdir -p gpurun_out/$OUT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err; echo "bench rc=$?" >> gpurun_out/$OUT/bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$OUT/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/$OUT/smoke.log
