#!/bin/bash
for F in "" "-DLMM_EMIT_BAND_MINB=7" "-DLMM_EMIT_BAND_MINB=6"; do
  export LMM_NVCC_EXTRA="$F"
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; continue; }
  for r in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$F] emit %.2f value %.4g' % (d['kernel_ms_per_step']['emit'], d['value']))"; done
done
