#!/bin/bash
# quick GPU check: build, selected tests, short bench (kernel times); TAG [pytest -k expr] [bench config]
TAG=$1; K=${2:-"parity or edges"}; CFG=${3:-octet100}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "$K" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 600 python bench.py --config $CFG --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["config"]["workload"][:40], "value %.4g %s" % (d["value"], d["unit"]), "ms/step %.2f" % d["ms_per_step"])
print({k: round(v, 2) for k, v in d["kernel_ms_per_step"].items()}, "emit frac %.3f" % d["roofline"]["frac"])
PY
tail -3 $O/bench.err
