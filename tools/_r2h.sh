set -x
OUT=${OUT:-r2h}; mkdir -p gpurun_out/$OUT
for cb in 1 2 4; do
AMVM_SCORE_CB=$cb AMVM_SCORE_THREADS=256 AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_nocomp.so timeout 300 python tools/scorer_sweep.py > gpurun_out/$OUT/nocomp_cb$cb.txt 2>&1
AMVM_SCORE_CB=$cb AMVM_SCORE_THREADS=256 timeout 300 python tools/scorer_sweep.py > gpurun_out/$OUT/full_cb$cb.txt 2>&1
done
