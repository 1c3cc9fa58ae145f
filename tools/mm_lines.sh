#!/bin/bash
# meta-mesh parts A/B/C (degree 9-12 bucket, octet40) per-source-line instruction counts
O=gpurun_out/mml; mkdir -p $O /tmp/mml
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="--steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --section SourceCounters --section LaunchStats --section SpeedOfLight --clock-control none --import-source on \
   --kernel-name-base demangled -k 'regex:metamesh_kernel<\(int\)[012], \(int\)32, \(int\)13,' -c 3 -o /tmp/mml/mm python bench.py --config octet40 $B > $O/ncu.log 2>&1
for p in 0 1 2; do
  python tools/ncu_lines.py /tmp/mml/mm.ncu-rep regex:metamesh_kernel@$p 60 $O/lines_p$p.csv > $O/lines_p$p.txt 2>&1
done
for p in 0 1 2; do python tools/ncu_sass.py /tmp/mml/mm.ncu-rep regex:metamesh_kernel@$p $O/sass_p$p.csv 2>> $O/sass.log; done
