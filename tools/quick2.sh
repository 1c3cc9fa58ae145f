#!/bin/bash
# quick GPU check: build, selected GPU tests (-k EXPR), default bench (+ optional config)
TAG=${1:-q}; K=${2:-}; CFG=${3:-}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
if [ -n "$K" ]; then timeout 1200 python -m pytest tests -q -m gpu -x -k "$K" > $O/pytest.log 2>&1; tail -3 $O/pytest.log; fi
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench.json 2> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench.json')); print('octet100', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3))"
if [ -n "$CFG" ]; then timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_$CFG.json 2>> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench_$CFG.json')); print('$CFG', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3), 'err', d['config'].get('error_nodes'))"; fi
