"""Per-phase cycle shares of the meta-mesh kernel (diagnostic build tools/liblmm_phase.so,
compiled with -DLMM_PHASE_TIMING).  Not part of the product path."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2405_15197_b200 import binding as B
B.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblmm_phase.so")
lib = B.load_library()
lib.lmm_debug_phase_cycles.argtypes = [C.c_void_p]
cfg = sys.argv[1] if len(sys.argv) > 1 else "octet40"
import re
fam, n = re.fullmatch(r"(octet|bcc|stoch)(\d+)", cfg).groups()
n = int(n)
if fam == "octet":
    lat = synth.graded_radii(synth.octet(n, n, n), 0.03, 0.06, 0)
elif fam == "bcc":
    lat = synth.bcc(n, n, n)
else:
    lat = synth.stochastic_window(n, n, 0, n - 1, seed=0)
xyz, ends, rend = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (lat.xyz, lat.ends, lat.r_end))
h = B.lmm_create(0, torch.cuda.current_stream().cuda_stream)
B.lmm_load_lattice(h, xyz, ends, rend)
B.lmm_build_metamesh(h)
torch.cuda.synchronize()
out = (C.c_ulonglong * 16)()
lib.lmm_debug_phase_cycles(out)
names = ["sides", "junctions", "clustering", "arcs(rest)", "drop+unref", "loops", "holes", "write",
         "arcs:pairs", "arcs:conic+int", "arcs:validity", "arcs:assemble", "live pairs", "p14", "p15", "p16"]
tot = sum(out)
print(cfg, lat.n_nodes, "nodes; cycles per node (lane-0 warps):", tot / lat.n_nodes)
for k, v in zip(names, out):
    if not v: continue
    print(f"  {k:12s} {100 * v / tot:5.1f}%  {v / lat.n_nodes:9.0f} cyc/node")
