set -x
OUT=${OUT:-r2g}; mkdir -p gpurun_out/$OUT
for cb in 2 4; do
AMVM_SCORE_CB=$cb AMVM_SCORE_THREADS=256 AMVM_LIBRARY=$PWD/paper_2508_13437_b200/libamvm_nocomp.so timeout 300 python tools/prof_scorer.py > gpurun_out/$OUT/nocomp_cb$cb.txt 2>&1
AMVM_SCORE_CB=$cb AMVM_SCORE_THREADS=256 timeout 300 python tools/prof_scorer.py > gpurun_out/$OUT/full_cb$cb.txt 2>&1
done
python - > gpurun_out/$OUT/copy.txt 2>&1 <<'PY'
import torch
x=torch.empty(64<<20,dtype=torch.uint8,device='cuda'); y=torch.empty_like(x); f=torch.empty(256<<20,dtype=torch.uint8,device='cuda')
xs=[torch.empty(8<<20,dtype=torch.float64,device='cuda') for _ in range(4)]
for _ in range(3): y.copy_(x)
import numpy as np
r=[]
for _ in range(10):
    f.zero_(); a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record(); y.copy_(x); b.record(); torch.cuda.synchronize(); r.append(a.elapsed_time(b))
print("copy 64MiB (128 MiB traffic) ms", np.median(r), "GB/s", 2*(64<<20)/np.median(r)/1e6)
r=[]
for _ in range(5):
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(16): s=xs[k%4].sum()
    b.record(); torch.cuda.synchronize(); r.append(a.elapsed_time(b)/16)
print("sum 64MiB cycled ms", np.median(r), "GB/s", (64<<20)/np.median(r)/1e6)
PY
