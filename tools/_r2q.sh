OUT=${OUT:-r2q}; mkdir -p gpurun_out/$OUT
BEST=0 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_active.avg --clock-control none -k regex:k_score_adj -c 6 python tools/scorer_sweep.py > gpurun_out/$OUT/ncu_sweep_best0.txt 2>&1
BEST=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_score_adj -c 6 python tools/scorer_sweep.py > gpurun_out/$OUT/ncu_sweep_best1.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"tma_read|ldg_read" -c 40 ./tools/ubench/read_bw > gpurun_out/$OUT/ncu_ubench.txt 2>&1
