OUT=${OUT:-r2j}; mkdir -p gpurun_out/$OUT
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_tl.so python tools/scorer_timeline.py > gpurun_out/$OUT/tl.txt 2>&1
python tools/scorer_sweep.py > gpurun_out/$OUT/sweep.txt 2>&1
timeout 600 python -m pytest tests/test_scoring.py tests/test_scoring_golden.py -x -q > gpurun_out/$OUT/pytest_score.log 2>&1; echo "rc=$?" >> gpurun_out/$OUT/pytest_score.log
python tools/prof_scorer.py > gpurun_out/$OUT/scorer.txt 2>&1
