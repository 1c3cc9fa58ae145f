"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel: total ms, launches, share."""
import csv, re, sys
from collections import defaultdict


def main(path, out, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        name = re.sub(r"^void ", "", r[ki])
        name = re.sub(r"\(.*$", "", name).replace("<unnamed>::", "")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}[r[ui]]
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    T = sum(tot.values())
    with open(out, "w") as f:
        f.write(f"# {title}\n# cold-cache serialised per-launch times: compare SHARES with the bench's event timing\n")
        f.write(f"{'kernel':60s} {'ms':>10s} {'launches':>8s} {'share':>7s}\n")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            f.write(f"{k[:60]:60s} {v:10.3f} {cnt[k]:8d} {100 * v / T:6.1f}%\n")


if __name__ == "__main__":
    main(*sys.argv[1:4])
