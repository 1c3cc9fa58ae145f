#!/bin/bash
# ncu --set full of one steady k_emit launch (octet100), report to gpurun_out/TAG; CE as $2
O=gpurun_out/${1:-ep}; mkdir -p $O; CE=${2:-1e-3}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREG:-k_emit} --launch-skip 2 -c 1 -o $O/emit_$CE \
  python bench.py --ce $CE --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > $O/ncu_$CE.log 2>&1; tail -2 $O/ncu_$CE.log
