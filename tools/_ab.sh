# A/B the given libraries (names under paper_2508_13437_b200/) on one box:
# a parity subset per library first, then interleaved bench runs.
D=gpurun_out/${AB_OUT:-ab}; mkdir -p $D
for L in "$@"; do
  echo "$L parity: $(AMVM_LIBRARY=$PWD/paper_2508_13437_b200/$L timeout 300 python -m pytest tests -m gpu -x -q -k 'named or chunked or overflow or small_solves' 2>&1 | tail -n 1)"
done
for rep in 1 2; do for L in "$@"; do
  AMVM_LIBRARY=$PWD/paper_2508_13437_b200/$L timeout 300 python bench.py --no-e2e --cpu-rows 1 --steps 4 > $D/$L.$rep.json 2>/dev/null
  python - $D/$L.$rep.json $L $rep <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print(sys.argv[2], sys.argv[3], round(d["value"] / 1e6, 1), "M/s", d["ms_steps"], "busy Gcyc", d["busy_gcycles_per_step"],
      {k: round(v, 3) for k, v in d["phase_share"].items() if v > 0.01})
PY
done; done
