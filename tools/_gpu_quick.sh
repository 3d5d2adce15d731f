# quick GPU check: parity suite + bench (no e2e) + per-phase probe
D=gpurun_out/${1:-q}; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -x -q > $D/pytest.log 2>&1; echo "pytest rc=$?" >> $D/pytest.log; tail -n 3 $D/pytest.log
timeout 600 python bench.py --no-e2e --cpu-rows 2 > $D/bench.json 2> $D/bench.err; echo "bench rc=$?"; cat $D/bench.json
