#!/bin/bash
# A/B of two prebuilt libraries (libab/liblmm_{base,new}.so) on one bench command
CMD=${1:-"python bench.py --config octet160 --ce 1e-4 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0"}
for r in 1 2; do for v in base new; do
  cp libab/liblmm_$v.so paper_2405_15197_b200/lib/liblmm.so
  $CMD 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', 'emit %.2f' % d['kernel_ms_per_step']['emit'], 'frac %.3f' % d['roofline']['frac'], 'value %.4g' % d['value'])"
done; done
cp libab/liblmm_new.so paper_2405_15197_b200/lib/liblmm.so
