#!/bin/bash
# round-2 checkpoint on a GPU box: build, all -m gpu tests, smoke, the bench line of every
# BASELINE config, ncu launch list of the default bench, ncu --set full summaries (k_emit at CE
# 1e-3 and 1e-2, the meta-mesh parts of the degree 9-12 and 24-31 buckets).  Reports stay on the
# box (too large); their text summaries come back in gpurun_out/TAG.
TAG=${1:-ck}
O=gpurun_out/$TAG; mkdir -p $O
R=/tmp/$TAG; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_octet100.json 2> $O/bench_octet100.err; tail -c 300 $O/bench_octet100.json
for c in bcc250 stoch290; do timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 1200 python bench.py --config octet160 --ce-sweep 1e-2,1e-3,1e-4 --steps 3 --warmup 3 > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 900 python bench.py --config octet100 --ce 1e-2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_octet100_ce1e-2.json 2> $O/bench_ce2.err
B="--steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_octet100.csv python bench.py $B > $O/ncu_list.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_stoch100.csv python bench.py --config stoch100 $B > $O/ncu_list2.log 2>&1
B="--steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_emit -c 1 -o $R/emit python bench.py $B > $O/ncu_emit.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_emit -c 1 -o $R/emit_ce2 python bench.py --ce 1e-2 $B > $O/ncu_emit2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:metamesh_kernel<\(int\)[012], \(int\)32, \(int\)13,' -c 3 -o $R/mm_octet python bench.py --config octet40 $B > $O/ncu_mm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:metamesh_kernel<\(int\)[012], \(int\)32, \(int\)32,' -c 3 -o $R/mm_stoch python bench.py --config stoch100 $B > $O/ncu_mm2.log 2>&1
T=$((1 << 28))
python tools/ncu_summary.py $R/emit.ncu-rep $O/emit_octet100_ncu.txt "k_emit, octet100 CE 1e-3 (one 2^28-triangle launch)" $T regex:k_emit
python tools/ncu_summary.py $R/emit_ce2.ncu-rep $O/emit_octet100_ce1e-2_ncu.txt "k_emit, octet100 CE 1e-2 (first launch)" "" regex:k_emit
for p in 0 1 2; do
  python tools/ncu_summary.py $R/mm_octet.ncu-rep $O/metamesh_part${p}_deg9-12_octet40_ncu.txt "meta-mesh part $p, degree 9-12 bucket, octet40" "" "regex:metamesh_kernel@$p"
  python tools/ncu_summary.py $R/mm_stoch.ncu-rep $O/metamesh_part${p}_deg24-31_stoch100_ncu.txt "meta-mesh part $p, degree 24-31 bucket, stoch100" "" "regex:metamesh_kernel@$p"
done
python tools/ncu_lines.py $R/emit.ncu-rep regex:k_emit 40 > $O/emit_lines.txt 2>&1
python tools/launch_summary.py $O/launches_octet100.csv $O/launches_octet100_summary.txt "ncu launch list, bench.py --steps 1 --warmup 1 (octet100 CE 1e-3)"
python tools/launch_summary.py $O/launches_stoch100.csv $O/launches_stoch100_summary.txt "ncu launch list, bench.py --config stoch100 --steps 1 --warmup 1"
ls $O
