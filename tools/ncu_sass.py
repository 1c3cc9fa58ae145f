"""Per-SASS-instruction executed counts of one kernel in an ncu report:
python tools/ncu_sass.py REPORT 'regex:NAME@SKIP' out.csv   (address, opcode text, warp-instructions, stall samples)"""
import csv, io, subprocess, sys


def main(rep, kern, outp):
    k, _, skip = kern.partition("@")
    out = subprocess.run(["ncu", "-i", rep, "-k", k, "--launch-skip", skip or "0", "--launch-count", "1", "--page",
                          "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
    hdr, rows = None, []
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Address":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[0]:
            rows.append((r[0], r[1].strip(), int(r[hdr.index("Instructions Executed")] or 0),
                         int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)))
    with open(outp, "w", newline="") as f:
        csv.writer(f).writerows(rows)
    print(len(rows), "sass rows", file=sys.stderr)


if __name__ == "__main__":
    main(*sys.argv[1:])
