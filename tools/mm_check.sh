#!/bin/bash
# meta-mesh change check: build, parity/edge GPU tests, meta-mesh ms on octet100 / stoch290
O=gpurun_out/${1:-mc}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu -k "${2:-parity or edges}" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for c in ${3:-octet100 stoch290}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/b_$c.json 2>/dev/null
  python - $O/b_$c.json $c <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    k=d["kernel_ms_per_step"]
    print(sys.argv[2], "value %.4g" % d["value"], "ms/step %.1f" % d["ms_per_step"], "mm %.2f" % k["metamesh"], "emit %.2f" % k["emit"], "err", d["config"].get("error_nodes"), "spill", d["config"].get("spilled_nodes"))
except Exception as e: print(sys.argv[2], "FAILED", e)
PY
done
