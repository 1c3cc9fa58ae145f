#!/bin/bash
# full checkpoint: all GPU tests, smoke, default bench, ncu launch list, emit + metamesh full captures
TAG=${1:-ck}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 600 $O/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $O/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_emit -c 1 -o $O/emit python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > $O/ncu_emit.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:metamesh|k_band' -c 11 -o $O/mm python bench.py --config octet40 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > $O/ncu_mm.log 2>&1
ls $O
