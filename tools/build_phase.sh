#!/bin/bash
# diagnostic build of liblmm with per-phase clock64 instrumentation of the meta-mesh kernel
# (tools/liblmm_phase.so), then the normal build again
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
cd $R
LMM_NVCC_EXTRA="-DLMM_PHASE_TIMING" python -c "import __graft_entry__ as g; g.build()" > /dev/null
cp paper_2405_15197_b200/lib/liblmm.so tools/liblmm_phase.so
python -c "import __graft_entry__ as g; g.build()" > /dev/null
