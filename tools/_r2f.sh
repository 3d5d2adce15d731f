set -x
OUT=${OUT:-r2f}; mkdir -p gpurun_out/$OUT
timeout 600 python -m pytest tests/test_scoring.py tests/test_scoring_golden.py -x -q > gpurun_out/$OUT/pytest_score.log 2>&1; echo "rc=$?" >> gpurun_out/$OUT/pytest_score.log
for cb in 1 2 4; do for nc in 512 256; do
AMVM_SCORE_CB=$cb AMVM_SCORE_THREADS=$nc timeout 300 python tools/prof_scorer.py > gpurun_out/$OUT/scorer_cb${cb}_nc${nc}.txt 2>&1
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_score_adj -c 1 -o gpurun_out/$OUT/score_adj env REPS=1 python tools/prof_scorer.py > gpurun_out/$OUT/ncu.log 2>&1; echo "ncu rc=$?"
