#!/bin/bash
# ncu --set full captures: TAG CONFIG KREGEX COUNT [extra bench args]
TAG=$1; CFG=$2; K=$3; C=${4:-1}; shift 4
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$K" -c $C -o $O/${CFG}_prof python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 "$@" > $O/ncu_$CFG.log 2>&1; tail -2 $O/ncu_$CFG.log
