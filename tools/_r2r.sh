OUT=${OUT:-r2r}; mkdir -p gpurun_out/$OUT
for cb in 2 4; do
BEST=0 AMVM_SCORE_CB=$cb AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_nocomp.so timeout 200 python tools/scorer_sweep.py > gpurun_out/$OUT/nocomp_cb$cb.txt 2>&1
BEST=0 AMVM_SCORE_CB=$cb AMVM_SCORE_THREADS=256 timeout 200 python tools/scorer_sweep.py > gpurun_out/$OUT/full256_cb$cb.txt 2>&1
done
