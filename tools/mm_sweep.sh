#!/bin/bash
# build variants (meta-mesh, count, emit ms): mm_sweep.sh "configs" "flags1" "flags2" ...
O=gpurun_out/mms; mkdir -p $O; CF=$1; shift
for F in "$@"; do
  export LMM_NVCC_EXTRA="$F"
  python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; continue; }
  for c in $CF; do
    timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null
    python - $O/b.json "[$F] $c" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d["kernel_ms_per_step"]
print(sys.argv[2], "value %.4g" % d["value"], "ms/step %.1f" % d["ms_per_step"], "mm %.2f" % k["metamesh"], "count %.2f" % k["count"], "emit %.2f" % k["emit"])
PY
  done
done
