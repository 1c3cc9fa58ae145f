O=gpurun_out/r1e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k stoch290 > $O/pytest_stoch.log 2>&1; tail -5 $O/pytest_stoch.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_emit -c 1 -o $O/emit_octet100 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > $O/ncu1.log 2>&1; tail -2 $O/ncu1.log
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_emit|metamesh|k_band' -c 12 -o $O/stoch120 python bench.py --config stoch120 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > $O/ncu2.log 2>&1; tail -2 $O/ncu2.log
