"""Key counters + top stalls + top source lines of one kernel in an ncu report.

    python tools/ncu_summary.py report.ncu-rep [--source N]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    nsrc = int(sys.argv[sys.argv.index("--source") + 1]) if "--source" in sys.argv else 0
    r = ncu_csv(rep, "raw")
    h, units = r[0], r[1]
    seen = set()
    for vals in r[2:]:  # one block per distinct kernel (first launch of each)
        d = dict(zip(h, vals))
        u = dict(zip(h, units))
        name = d.get("Kernel Name", "?")[:100]
        if name in seen:
            continue
        seen.add(name)
        print("kernel:", name)
        for k in KEYS:
            if k in d:
                print("  %-75s %s %s" % (k, d[k], u.get(k, "")))
        st = [(float(v), n) for n, v in d.items()
              if "average_warps_issue_stalled" in n and "per_issue_active" in n and v]
        print("  top stalls (warps per issue):")
        for v, n in sorted(st, reverse=True)[:8]:
            print("    %.3f %s" % (v, n.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", "")))
    if nsrc:
        rows = ncu_csv(rep, "source", ["--print-source", "sass"])
        hdr = rows[1]
        idx = {k: i for i, k in enumerate(hdr)}
        data = rows[2:]

        def f(row, k):
            try:
                return float(row[idx[k]].replace(",", ""))
            except (ValueError, KeyError, IndexError):
                return 0.0
        key = "Warp Stall Sampling (All Samples)"
        tot = sum(f(x, key) for x in data) or 1.0
        print("  top stall-sampled SASS:")
        for x in sorted(data, key=lambda x: -f(x, key))[:nsrc]:
            print("    %5.1f%%  %s" % (100 * f(x, key) / tot, x[idx["Source"]].strip()[:90]))


if __name__ == "__main__":
    main()
