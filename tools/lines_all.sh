#!/bin/bash
# full per-line/SASS instruction tables of k_emit (CE 1e-3, 1e-2) and the meta-mesh parts
# (octet40, degree 9-12 bucket), plus one default bench line
mkdir -p gpurun_out/la
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/la/build.log 2>&1 || exit 1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/la/bench.json 2> gpurun_out/la/bench.err
bash tools/emit_lines.sh
bash tools/mm_lines.sh
ls -la gpurun_out/el gpurun_out/mml
