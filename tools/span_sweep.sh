#!/bin/bash
# CTA-window emit: build variants x window sizes (emit ms); TAG "flags1" "flags2" ...
O=gpurun_out/$1; shift; mkdir -p $O
i=0
for F in "$@"; do
  i=$((i+1)); export LMM_NVCC_EXTRA="$F"
  python -c "import __graft_entry__ as g; g.build()" > $O/build$i.log 2>&1 || { echo "build $i failed"; continue; }
  [ $i = 1 ] && { timeout 900 python -m pytest tests -x -q -m gpu -k "parity or edges" > $O/pytest.log 2>&1; tail -1 $O/pytest.log; }
  for ce in 1e-3 1e-2; do for pcw in ${PCWS:-768 1024}; do
    LMM_EMIT_PATH=1 LMM_SPCW=$pcw timeout 300 python bench.py --ce $ce --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/b$i_${ce}_$pcw.json 2>/dev/null
    python - $O/b$i_${ce}_$pcw.json "[$F] ce $ce pcw $pcw" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "value %.4g" % d["value"], "emit %.2f ms" % d["kernel_ms_per_step"]["emit"], "frac %.3f" % d["roofline"]["frac"])
except Exception as e: print(sys.argv[2], "FAILED", e)
PY
  done; done
done
