OUT=${OUT:-r2l}; mkdir -p gpurun_out/$OUT
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_tl.so python tools/scorer_timeline.py > gpurun_out/$OUT/tl.txt 2>&1
AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_tlnc.so python tools/scorer_timeline.py > gpurun_out/$OUT/tlnc.txt 2>&1
AMVM_SCORE_CB=1 AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_tl.so python tools/scorer_timeline.py > gpurun_out/$OUT/tl_cb1.txt 2>&1
