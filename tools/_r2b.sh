set -x
OUT=${OUT:-r2b}; mkdir -p gpurun_out/$OUT
timeout 600 python -m pytest tests/test_scoring.py tests/test_scoring_golden.py -x -q > gpurun_out/$OUT/pytest_score.log 2>&1; echo "rc=$?" >> gpurun_out/$OUT/pytest_score.log
timeout 300 python tools/prof_scorer.py > gpurun_out/$OUT/scorer.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_score_adj -c 1 -o gpurun_out/$OUT/score_adj env REPS=1 python tools/prof_scorer.py > gpurun_out/$OUT/ncu.log 2>&1; echo "ncu rc=$?"
