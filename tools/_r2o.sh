OUT=${OUT:-r2o}; mkdir -p gpurun_out/$OUT
for t in tl tlr tlf; do AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_$t.so timeout 120 python tools/scorer_timeline.py > gpurun_out/$OUT/$t.txt 2>&1; done
