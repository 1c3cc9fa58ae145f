#!/bin/bash
# CTA-window emit check: build, parity/edge GPU tests, then emit time per window size / path
O=gpurun_out/${1:-sc}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu -k "${2:-parity or edges}" > $O/pytest.log 2>&1; tail -5 $O/pytest.log
for ce in 1e-3 1e-2; do for cfg in ${3:-"0:768" "1:512" "1:768" "1:1024"}; do
  path=${cfg%%:*}; pcw=${cfg##*:}
  export LMM_EMIT_PATH=$path LMM_SPCW=$pcw
  timeout 300 python bench.py --ce $ce --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/b_${ce}_${path}_$pcw.json 2> $O/b_${ce}_${path}_$pcw.err
  python - $O/b_${ce}_${path}_$pcw.json "ce $ce path $path pcw $pcw" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "value %.4g" % d["value"], "ms/step %.2f" % d["ms_per_step"], "emit %.2f ms" % d["kernel_ms_per_step"]["emit"], "frac %.3f" % d["roofline"]["frac"])
except Exception as e: print(sys.argv[2], "FAILED", e)
PY
done; done
unset LMM_EMIT_PATH LMM_SPCW
