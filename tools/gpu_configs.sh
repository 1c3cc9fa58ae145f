#!/bin/bash
# Bench lines of the non-default BASELINE configs (1 GPU each); outputs under gpurun_out/$TAG.
TAG=${1:-cfg}; shift
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { cat $O/build.log; exit 1; }
for c in ${*:-bcc250 stoch290 sweep}; do
  case $c in
    sweep) timeout 1200 python bench.py --config octet160 --ce-sweep 1e-2,1e-3,1e-4 --steps 3 --warmup 3 > $O/bench_sweep.json 2> $O/bench_sweep.err ;;
    *)     timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err ;;
  esac
  echo "== $c rc=$?"; tail -c 1500 $O/bench_$c.json; tail -3 $O/bench_$c.err
done
