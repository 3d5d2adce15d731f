set -x
OUT=${OUT:-r1f}; mkdir -p gpurun_out/$OUT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${OUT:-r1f}/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${OUT:-r1f}/pytest.log
timeout 900 python bench.py > gpurun_out/${OUT:-r1f}/bench.json 2> gpurun_out/${OUT:-r1f}/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${OUT:-r1f}/bench_ref.json 2> gpurun_out/${OUT:-r1f}/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${OUT:-r1f}/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --cpu-rows 2 > gpurun_out/${OUT:-r1f}/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/${OUT:-r1f}/ksolve python bench.py --steps 1 --warmup 3 --no-e2e --cpu-rows 2 > gpurun_out/${OUT:-r1f}/ncu_full.log 2>&1; echo "ncu2 rc=$?"
