#!/bin/bash
# per-phase cycle profile of the meta-mesh kernel for csrc variants: phase_run.sh "configs" VARIANT...
O=gpurun_out/phase; mkdir -p $O
CFGS=$1; shift
SRC=paper_2405_15197_b200/csrc
mkdir -p /tmp/ph_orig && cp $SRC/*.cu $SRC/*.cuh $SRC/*.h /tmp/ph_orig/
for V in "$@"; do
  cp /tmp/ph_orig/* $SRC/; cp tools/ab_variants/$V/* $SRC/
  LMM_NVCC_EXTRA="-DLMM_PHASE_TIMING" python -c "import __graft_entry__ as g; g.build()" > $O/build_$V.log 2>&1 || { echo build $V failed; continue; }
  cp paper_2405_15197_b200/lib/liblmm.so tools/liblmm_phase.so
  for c in $CFGS; do echo "== $V"; timeout 300 python tools/phase_profile.py $c; done
done
cp /tmp/ph_orig/* $SRC/
python -c "import __graft_entry__ as g; g.build()" > $O/build_final.log 2>&1
