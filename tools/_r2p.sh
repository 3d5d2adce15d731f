OUT=${OUT:-r2p}; mkdir -p gpurun_out/$OUT
timeout 300 python -m pytest tests/test_scoring.py tests/test_scoring_golden.py -x -q > gpurun_out/$OUT/pytest_score.log 2>&1; echo "rc=$?" >> gpurun_out/$OUT/pytest_score.log
for B in 1 0; do
BEST=$B AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_tl.so timeout 120 python tools/scorer_timeline.py > gpurun_out/$OUT/tl_best$B.txt 2>&1
BEST=$B timeout 200 python tools/scorer_sweep.py > gpurun_out/$OUT/sweep_best$B.txt 2>&1
BEST=$B AMVM_SCORE_CB=4 timeout 200 python tools/scorer_sweep.py > gpurun_out/$OUT/sweep_cb4_best$B.txt 2>&1
done
