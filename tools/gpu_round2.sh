set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputest.log 2>&1
tail -40 gpurun_out/gputest.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/bench.log
