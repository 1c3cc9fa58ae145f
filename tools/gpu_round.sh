#!/bin/bash
# One GPU session: build, gpu tests, smoke, bench (N=1 default), ncu launch list + full captures.
# usage: tools/gpu_round.sh TAG [tests|bench|ncu ...]
set -x
TAG=${1:-r1}; shift
WHAT=${*:-tests bench ncu}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { cat $O/build.log; exit 1; }
for w in $WHAT; do case $w in
tests) timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
       timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log ;;
bench) timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 3000 $O/bench.json; tail -5 $O/bench.err ;;
ncu)   timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
          python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $O/ncu_bench.log 2>&1
       timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:k_emit|metamesh_kernel|k_band_count|k_band_merge' \
          -c 8 -o $O/full python bench.py --config octet40 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > $O/ncu_full.log 2>&1
       tail -3 $O/ncu_full.log ;;
esac; done
