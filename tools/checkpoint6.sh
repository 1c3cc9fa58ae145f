#!/bin/bash
# round-2 checkpoint f: build, smoke, all -m gpu tests, the bench line of every BASELINE
# config, the reference arm, 2-rank functional runs of the multi-rank path on one GPU (gloo),
# and the ncu launch list + k_emit summary of the default bench.
TAG=${1:-ck}
O=gpurun_out/$TAG; mkdir -p $O
R=/tmp/$TAG; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_octet100.json 2> $O/bench_octet100.err; tail -c 400 $O/bench_octet100.json
for c in bcc250 stoch290; do timeout 1500 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 1500 python bench.py --config octet160 --ce-sweep 1e-2,1e-3,1e-4 --steps 3 --warmup 3 > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 900 python bench.py --config octet100 --ce 1e-2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_octet100_ce1e-2.json 2> $O/bench_ce2.err
LMM_EMIT_PATH=1 timeout 1500 python bench.py --config stoch290 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_stoch290_span.json 2> $O/bench_stoch290_span.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
for c in octet40 bcc40 stoch40; do
  LMM_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus 2 --config $c --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $O/bench_2rank_$c.json 2> $O/bench_2rank_$c.err
done
B="--steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_octet100.csv python bench.py $B > $O/ncu_list.log 2>&1
B="--steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_emit -c 1 -o $R/emit python bench.py $B > $O/ncu_emit.log 2>&1
python tools/ncu_summary.py $R/emit.ncu-rep $O/emit_octet100_ncu.txt "k_emit, octet100 CE 1e-3 (one 2^28-triangle launch)" $((1 << 28)) regex:k_emit
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_emit_span -c 1 --launch-skip 2 -o $R/emit_span python bench.py --ce 1e-2 $B > $O/ncu_emit_span.log 2>&1
python tools/ncu_summary.py $R/emit_span.ncu-rep $O/emit_span_octet100_ce1e-2_ncu.txt "k_emit_span, octet100 CE 1e-2 (one 2^28-triangle launch)" $((1 << 28)) regex:k_emit_span
python tools/launch_summary.py $O/launches_octet100.csv $O/launches_octet100_summary.txt "ncu launch list, bench.py --steps 1 --warmup 1 (octet100 CE 1e-3)"
ls $O
