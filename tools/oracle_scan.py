#!/usr/bin/env python
"""Scan every node of a synthetic workload with the CPU oracle (test infrastructure: the
oracle's status of each node, nothing kept), in parallel worker processes.

    python tools/oracle_scan.py stoch290 [--procs 8] [--bits 32] [--out gpurun_out/scan.npz]

Prints the status histogram and the first nodes in error; --out saves (node, status) of
every node in error.  Used to locate nodes the model refuses at full size."""
import argparse
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

_LAT = None


def _work(args):
    lo, hi, bits = args
    import oracle
    orc = oracle.Oracle(_LAT.xyz, _LAT.node_r, _LAT.ends, bits)
    st, _ = orc.scan(np.arange(lo, hi, dtype=np.int64))
    bad = np.flatnonzero(st) + lo
    return bad, st[bad - lo]


def main():
    global _LAT
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--bits", type=int, default=32)
    ap.add_argument("--chunk", type=int, default=200_000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import bench
    import oracle
    oracle.build_oracle()
    t0 = time.time()
    _LAT, _, _ = bench.make_config(a.config)
    print(f"{a.config}: {_LAT.n_nodes} nodes, {_LAT.n_struts} struts, generated in {time.time() - t0:.1f} s", flush=True)
    t0 = time.time()
    jobs = [(lo, min(lo + a.chunk, _LAT.n_nodes), a.bits) for lo in range(0, _LAT.n_nodes, a.chunk)]
    bad, st = [], []
    with mp.get_context("fork").Pool(a.procs) as pool:
        for i, (b, s) in enumerate(pool.imap(_work, jobs)):
            bad.append(b)
            st.append(s)
            if i % 20 == 0:
                print(f"  {i + 1}/{len(jobs)} chunks, {time.time() - t0:.0f} s, errors so far {sum(len(x) for x in bad)}", flush=True)
    bad = np.concatenate(bad)
    st = np.concatenate(st)
    print(f"scanned in {time.time() - t0:.1f} s with {a.procs} processes")
    codes, cnt = np.unique(st, return_counts=True)
    print("errors:", {oracle.ORC_STATUS[int(c)]: int(k) for c, k in zip(codes, cnt)})
    print("first:", list(zip(bad[:20].tolist(), st[:20].tolist())))
    if a.out:
        np.savez(a.out, node=bad, status=st)


if __name__ == "__main__":
    main()
