#!/bin/bash
# k_emit per-source-line instruction counts and stall samples (octet100 CE 1e-3 and 1e-2)
O=gpurun_out/el; mkdir -p $O /tmp/el
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for ce in 1e-3 1e-2; do
  timeout 900 ncu --section SourceCounters --section LaunchStats --section SpeedOfLight --clock-control none --import-source on \
     -k regex:k_emit -c 1 -o /tmp/el/emit_$ce python bench.py --ce $ce --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu_$ce.log 2>&1
  python tools/ncu_lines.py /tmp/el/emit_$ce.ncu-rep regex:k_emit 60 $O/lines_$ce.csv > $O/lines_$ce.txt 2>&1
done
python tools/ncu_sass.py /tmp/el/emit_1e-3.ncu-rep regex:k_emit $O/sass_1e-3.csv 2>> $O/sass.log
