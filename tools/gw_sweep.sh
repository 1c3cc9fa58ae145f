#!/bin/bash
# CTA-window emit: group width / window entries build variants, emit ms at CE 1e-3 and 1e-2
O=gpurun_out/gw; mkdir -p $O
for F in "" "-DLMM_SPAN_GW=48 -DLMM_SPAN_SEC=96" "-DLMM_SPAN_GW=48"; do
  export LMM_NVCC_EXTRA="$F"
  python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; continue; }
  [ -n "$F" ] && { timeout 900 python -m pytest tests -q -x -m gpu -k "emit_paths" 2>&1 | tail -1; }
  for ce in 1e-3 1e-2; do for pcw in 768 1280; do
    LMM_EMIT_PATH=1 LMM_SPCW=$pcw timeout 300 python bench.py --ce $ce --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$F] ce $ce pcw $pcw emit %.2f' % d['kernel_ms_per_step']['emit'])"
  done; done
done
