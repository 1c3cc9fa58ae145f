#!/bin/bash
# span-path check: build, parity/edge GPU tests (-x), then emit time per point-cache size
O=gpurun_out/${1:-sp}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu -k "${2:-parity or edges}" > $O/pytest.log 2>&1; tail -5 $O/pytest.log
for ce in 1e-3 1e-2; do for wc in ${3:-0 256 288 320 384}; do
  if [ $wc = 0 ]; then unset LMM_WCAP; else export LMM_WCAP=$wc; fi
  timeout 300 python bench.py --ce $ce --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/bench_${ce}_$wc.json 2> $O/bench_${ce}_$wc.err
  python - $O/bench_${ce}_$wc.json $ce $wc <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("ce", sys.argv[2], "wcap", sys.argv[3], "value %.4g" % d["value"], "ms/step %.2f" % d["ms_per_step"], "emit %.2f ms" % d["kernel_ms_per_step"]["emit"], "frac %.3f" % d["roofline"]["frac"])
except Exception as e: print("ce", sys.argv[2], "wcap", sys.argv[3], "FAILED", e)
PY
done; done
unset LMM_WCAP
