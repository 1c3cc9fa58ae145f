#!/bin/bash
# build variants (LMM_NVCC_EXTRA) and bench each: sweep.sh TAG "configs" "flags1" "flags2" ...
TAG=$1; CFGS=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
i=0
for F in "$@"; do
  i=$((i+1))
  export LMM_NVCC_EXTRA="$F"
  python -c "import __graft_entry__ as g; g.build()" > $O/build$i.log 2>&1 || { echo "build $i failed"; tail -5 $O/build$i.log; continue; }
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "metamesh" > $O/pytest$i.log 2>&1; echo "== [$F] $(tail -1 $O/pytest$i.log)"
  for c in $CFGS; do
    timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/bench${i}_$c.json 2> $O/bench${i}_$c.err
    python - $O/bench${i}_$c.json $c <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("  ", sys.argv[2], "%.4g %s" % (d["value"], d["unit"]), "ms/step %.2f" % d["ms_per_step"], {k: round(v, 2) for k, v in d["kernel_ms_per_step"].items()})
except Exception as e:
    print("  ", sys.argv[2], "failed", e)
PY
  done
done
