OUT=${OUT:-r2u}; mkdir -p gpurun_out/$OUT
timeout 300 python tools/prof_c5.py 592 20 > gpurun_out/$OUT/prof_c5.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/$OUT/ksolve python tools/prof_c5.py 296 10 > gpurun_out/$OUT/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/$OUT/ncu.log
