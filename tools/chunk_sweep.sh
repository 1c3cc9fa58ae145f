for L in 28 27 29 30 28; do
  LMM_BENCH_CHUNK_LOG2=$L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ch.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ch.json').read().strip().splitlines()[-1]); print($L, 'value %.4g' % d['value'], 'emit %.2f' % d['kernel_ms_per_step']['emit'], 'frac %.4f' % d['roofline']['frac'], d['roofline']['launches'])"
done
