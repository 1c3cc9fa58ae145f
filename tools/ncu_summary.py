"""Summarise an ncu --set full report (run here, with ncu -i) into a short text file."""
import csv, io, subprocess, sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Avg. Active Threads Per Warp", "Achieved Active Warps Per SM", "Theoretical Occupancy",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Limit Registers", "Block Limit Shared Mem",
        "No Eligible", "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum",
       "smsp__thread_inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__thread_inst_executed_per_inst_executed.ratio",
       "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum"]


KFILTER = []


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *KFILTER, *args], capture_output=True, text=True).stdout


def main(rep, out, title, units=None, kernel=None):
    """kernel: optional ncu -k filter (e.g. 'regex:k_emit') selecting one kernel of the report."""
    KFILTER[:] = []
    if kernel:   # "regex:NAME" or "regex:NAME@SKIP" (SKIP-th matching launch)
        k, _, skip = kernel.partition("@")
        KFILTER[:] = ["-k", k, "--launch-skip", skip or "0", "--launch-count", "1"]
    det = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    hdr = det[0]
    rows = [dict(zip(hdr, r)) for r in det[1:]]
    name = rows[0].get("Kernel Name", "?") if rows else "?"
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    rd = dict(zip(raw[0], raw[2])) if len(raw) > 2 else {}
    ru = dict(zip(raw[0], raw[1])) if len(raw) > 1 else {}
    sass = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source=sass"))))
    stalls = {}
    if len(sass) > 2:
        h = sass[1]
        cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
        body = [r for r in sass[2:] if len(r) == len(h)]
        tot = {c: sum(int(r[h.index(c)]) if r[h.index(c)].isdigit() else 0 for r in body) for c in cols}
        T = sum(tot.values()) or 1
        stalls = {c: 100 * v / T for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]}
    with open(out, "w") as f:
        f.write(f"# {title}\n# report: {rep}\n# kernel: {name}\n\n")
        seen = set()
        for r in rows:
            k = r.get("Metric Name")
            if k in KEYS and k not in seen:
                seen.add(k)
                f.write(f"{k:40s} {r.get('Metric Value')} {r.get('Metric Unit')}\n")
        f.write("\n")
        for k in RAW:
            if k in rd:
                f.write(f"{k:40s} {rd[k]} {ru.get(k, '')}\n")
        # north_star's meta-mesh evidence: global sectors per request (coalescing) and warp
        # execution efficiency (active threads per executed instruction / 32)
        for op in ("ld", "st"):
            sk, rk = f"l1tex__t_sectors_pipe_lsu_mem_global_op_{op}.sum", f"l1tex__t_requests_pipe_lsu_mem_global_op_{op}.sum"
            try:
                sec, req = float(rd[sk].replace(",", "")), float(rd[rk].replace(",", ""))
                f.write(f"global {op} sectors per request             {sec / req if req else 0:.2f}\n")
            except (KeyError, ValueError):
                pass
        try:
            r = float(rd["smsp__thread_inst_executed_per_inst_executed.ratio"].replace(",", ""))
            f.write(f"warp execution efficiency                {100 * r / 32:.1f} %\n")
        except (KeyError, ValueError):
            pass
        if units:
            try:
                rbytes = float(rd["dram__bytes_read.sum"]) * (1e9 if "G" in ru["dram__bytes_read.sum"] else 1e6)
                wbytes = float(rd["dram__bytes_write.sum"]) * (1e9 if "G" in ru["dram__bytes_write.sum"] else 1e6)
                f.write(f"\nunits per launch                         {units:.6g}\n")
                f.write(f"DRAM bytes per unit (read+write)         {(rbytes + wbytes) / units:.2f}\n")
            except (KeyError, ValueError):
                pass
        f.write("\nwarp stall reasons (share of samples):\n")
        for c, v in stalls.items():
            f.write(f"  {c:28s} {v:5.1f}%\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4] else None,
         sys.argv[5] if len(sys.argv) > 5 else None)
