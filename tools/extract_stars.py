#!/usr/bin/env python
"""Cut the stars (node + incident struts + far nodes, exact binary32 coordinates, strut order
and end orientation preserved) of given nodes out of a synthetic workload into a JSON fixture,
so a node found at full size can be meta-meshed alone (its meta-mesh depends on nothing else).

    python tools/extract_stars.py stoch290 1853282 3667395 ... --out tests/golden/x.json
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def star_of(lat, n):
    s = np.flatnonzero((lat.ends[:, 0] == n) | (lat.ends[:, 1] == n))   # ascending strut id
    far = np.where(lat.ends[s, 0] == n, lat.ends[s, 1], lat.ends[s, 0])
    xyz = np.concatenate([lat.xyz[[n]], lat.xyz[far]]).astype(np.float32)
    r = np.concatenate([lat.node_r[[n]], lat.node_r[far]]).astype(np.float32)
    # keep each strut's orientation (i0 -> i1): the strut frame of the loops depends on it
    ends = [[0, k + 1] if lat.ends[si, 0] == n else [k + 1, 0] for k, si in enumerate(s)]
    return dict(node=int(n), xyz=xyz.astype(np.float64).tolist(), r=r.astype(np.float64).tolist(), ends=ends)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("nodes", type=int, nargs="+")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    import bench
    lat, _, desc = bench.make_config(a.config)
    stars = [star_of(lat, n) for n in a.nodes]
    json.dump(dict(source=f"{a.config}: {desc}", note=a.note, stars=stars), open(a.out, "w"), indent=1)
    print(f"wrote {len(stars)} stars to {a.out}")


if __name__ == "__main__":
    main()
