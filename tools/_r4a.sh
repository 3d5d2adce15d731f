#!/bin/bash
# pairwise-sum stacks in smem + scorer PDL: parity suite, scorer sweep with PDL on/off
mkdir -p gpurun_out/r4a
python -c "import torch; print(torch.cuda.get_device_name())"
for p in 1 0; do
  AMVM_SCORE_PDL=$p timeout 300 python tools/scorer_sweep.py > gpurun_out/r4a/sweep_pdl$p.log 2>&1
done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r4a/pytest.log 2>&1
echo "pytest exit $?"
tail -3 gpurun_out/r4a/pytest.log
cat gpurun_out/r4a/sweep_pdl*.log
