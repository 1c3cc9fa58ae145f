#!/bin/bash
for F in "" "-DLMM_EMIT_BAND_MINB=7"; do
  export LMM_NVCC_EXTRA="$F"
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; continue; }
  [ -n "$F" ] && { timeout 900 python -m pytest tests -q -x -m gpu -k "parity or emit_paths or edges" 2>&1 | tail -1; }
  for a in "--config bcc250" "--config stoch290" "--config octet160 --ce 1e-4" "--ce 1e-2"; do
    timeout 600 python bench.py $a --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$F] $a emit %.2f value %.4g' % (d['kernel_ms_per_step']['emit'], d['value']))"
  done
done
