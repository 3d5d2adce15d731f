#!/bin/bash
# lane-per-pair find_candidates: parity suite, C1/C2 phases (pairs vs i-groups), C5 bench, scorer PDL A/B
OUT=${OUT:-r4b}; mkdir -p gpurun_out/$OUT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/$OUT/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$OUT/pytest.log
tail -2 gpurun_out/$OUT/pytest.log
python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps_pairs.txt 2>&1
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_nopairs.so python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps_nopairs.txt 2>&1
FCPROF=1 AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_fcprof.so python tools/phase_single.py c1 c2 > gpurun_out/$OUT/ps_fcprof.txt 2>&1
for p in 0 1 0 1; do
  echo "PDL=$p" >> gpurun_out/$OUT/sweep.log
  AMVM_SCORE_PDL=$p timeout 300 python tools/scorer_sweep.py >> gpurun_out/$OUT/sweep.log 2>&1
done
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-legs > gpurun_out/$OUT/bench.json 2> gpurun_out/$OUT/bench.err
cat gpurun_out/$OUT/ps_*.txt
