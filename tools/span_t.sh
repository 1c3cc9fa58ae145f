#!/bin/bash
# CTA-window emit: threads per CTA x window size
O=gpurun_out/st; mkdir -p $O
for T in 128 256; do
  export LMM_NVCC_EXTRA="-DLMM_SPAN_T=$T"
  python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; continue; }
  [ $T = 256 ] && { timeout 900 python -m pytest tests -q -x -m gpu -k "emit_paths or parity" 2>&1 | tail -1; }
  for ce in 1e-2 1e-3; do for pcw in ${PCWS:-768 1536}; do
    LMM_EMIT_PATH=1 LMM_SPCW=$pcw timeout 300 python bench.py --ce $ce --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('T $T pcw $pcw ce $ce', 'emit %.2f' % d['kernel_ms_per_step']['emit'], 'frac %.3f' % d['roofline']['frac'])"
  done; done
done
