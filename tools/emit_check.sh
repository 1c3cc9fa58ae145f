#!/bin/bash
# emit team-width check: parity tests with all bands on half-warp teams, with none, and the
# default; then A/B benches (CE 1e-2 and 1e-3) against tools/ab_variants/base
O=gpurun_out/${1:-ec}; mkdir -p $O
for F in "-DLMM_EMIT_HALF_BELOW=1e9" "-DLMM_EMIT_HALF_BELOW=0" ""; do
  export LMM_NVCC_EXTRA="$F"
  python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -5 $O/build.log; exit 1; }
  timeout 900 python -m pytest tests -q -m gpu -x -k "triangulation or ranges or sweep or remesh or edges or virtual or random" > $O/pytest.log 2>&1
  echo "[$F] $(tail -1 $O/pytest.log)"
done
unset LMM_NVCC_EXTRA
for V in base new; do
  mkdir -p /tmp/abo; cp paper_2405_15197_b200/csrc/* /tmp/abo/
  [ "$V" = base ] && cp tools/ab_variants/base/* paper_2405_15197_b200/csrc/
  python -c "import __graft_entry__ as g; g.build()" > $O/build_$V.log 2>&1
  for ce in 1e-2 1e-3; do
    timeout 600 python bench.py --ce $ce --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $O/b_${V}_$ce.json 2>/dev/null
    python -c "
import json; d=json.loads(open('$O/b_${V}_$ce.json').read().strip().splitlines()[-1]); print('$V ce $ce', round(d['ms_per_step'],2), 'emit', round(d['kernel_ms_per_step']['emit'],2), 'frac', round(d['roofline']['frac'],3))"
  done
  cp /tmp/abo/* paper_2405_15197_b200/csrc/
done
