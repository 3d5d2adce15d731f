OUT=${OUT:-r2m}; mkdir -p gpurun_out/$OUT
timeout 600 python -m pytest tests/test_scoring.py tests/test_scoring_golden.py -x -q > gpurun_out/$OUT/pytest_score.log 2>&1; echo "rc=$?" >> gpurun_out/$OUT/pytest_score.log
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_tl.so timeout 120 python tools/scorer_timeline.py > gpurun_out/$OUT/tl.txt 2>&1
AMVM_SCORE_CB=4 AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_tl.so timeout 120 python tools/scorer_timeline.py > gpurun_out/$OUT/tl_cb4.txt 2>&1
for cb in 1 2 4; do AMVM_SCORE_CB=$cb timeout 200 python tools/scorer_sweep.py > gpurun_out/$OUT/sweep_cb$cb.txt 2>&1; done
AMVM_SCORE_THREADS=256 timeout 200 python tools/scorer_sweep.py > gpurun_out/$OUT/sweep_nc256.txt 2>&1
timeout 200 python tools/prof_scorer.py > gpurun_out/$OUT/scorer.txt 2>&1
