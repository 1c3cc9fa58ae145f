#!/bin/bash
# round-2 profiling pass: ncu --set full (with source) of the meta-mesh parts (octet40: degree
# 9-12 bucket), k_emit and the count kernels of the default bench.  PART=stoch: the two top
# degree buckets of stoch100 instead.  Keep gpurun_out under 64 MiB.
TAG=${1:-r2p}; PART=${2:-octet}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
B="--steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
if [ "$PART" = octet ]; then
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:metamesh_kernel<\(int\)[012], \(int\)32, \(int\)13,' -c 3 -o $O/mm_octet40 python bench.py --config octet40 $B > $O/ncu_mm_octet40.log 2>&1
[ -n "$TRI" ] && timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_emit|k_band_merge|k_ring_count' -c 3 -o $O/tri_octet100 python bench.py $B > $O/ncu_tri.log 2>&1
else
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:metamesh_kernel<\(int\)[012], \(int\)32, \(int\)(24|32),' -c 6 -o $O/mm_stoch100 python bench.py --config stoch100 $B > $O/ncu_mm_stoch100.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_stoch100.csv python bench.py --config stoch100 $B > $O/ncu_list.log 2>&1
fi
ls -la $O
