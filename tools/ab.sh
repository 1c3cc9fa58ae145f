#!/bin/bash
# A/B on one box: ab.sh TAG "configs" VARIANT... ; each VARIANT is a directory of replacement
# csrc files (tools/ab_variants/NAME); builds each, benches each config, restores the tree.
TAG=$1; CFGS=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
SRC=paper_2405_15197_b200/csrc
mkdir -p /tmp/ab_orig && cp $SRC/*.cu $SRC/*.cuh $SRC/*.h /tmp/ab_orig/
for V in "$@"; do
  cp /tmp/ab_orig/* $SRC/
  cp tools/ab_variants/$V/* $SRC/
  python -c "import __graft_entry__ as g; g.build()" > $O/build_$V.log 2>&1 || { echo "build $V failed"; tail -5 $O/build_$V.log; continue; }
  for c in $CFGS; do
    timeout 600 python bench.py --config $c --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/bench_${V}_$c.json 2> $O/bench_${V}_$c.err
    python - $O/bench_${V}_$c.json $c $V <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("  ", sys.argv[3], sys.argv[2], "ms/step %.2f" % d["ms_per_step"], {k: round(v, 2) for k, v in d["kernel_ms_per_step"].items()})
except Exception as e:
    print("  ", sys.argv[3], sys.argv[2], "failed", e)
PY
  done
done
cp /tmp/ab_orig/* $SRC/
