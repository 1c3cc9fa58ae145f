"""Per-source-line hot spots of one kernel in an ncu report (cuda,sass view):
python tools/ncu_lines.py REPORT 'regex:NAME@SKIP' [top] [full.csv]"""
import csv, io, subprocess, sys


def main(rep, kern, top=40, full=None):
    k, _, skip = kern.partition("@")
    out = subprocess.run(["ncu", "-i", rep, "-k", k, "--launch-skip", skip or "0", "--launch-count", "1", "--page",
                          "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
    rows, fname, hdr = [], "?", None
    for r in csv.reader(io.StringIO(out)):
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[0]:
            ie = int(r[hdr.index("Instructions Executed")] or 0)
            sm = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            rows.append((fname, int(r[0]), ie, sm, r[1].strip()[:90]))
    if full:   # every line: file, line, warp-instructions, stall samples, source
        with open(full, "w", newline="") as f:
            csv.writer(f).writerows(rows)
    ti = sum(x[2] for x in rows) or 1
    ts = sum(x[3] for x in rows) or 1
    print(f"total warp-instructions {ti}, stall samples {ts}")
    for f, ln, ie, sm, src in sorted(rows, key=lambda x: -x[3])[:int(top)]:
        print(f"{f}:{ln:<5d} inst {100 * ie / ti:5.1f}%  samples {100 * sm / ts:5.1f}%  {src}")


if __name__ == "__main__":
    main(*sys.argv[1:])
