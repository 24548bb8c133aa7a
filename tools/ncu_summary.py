"""Summaries of ncu reports: key metrics per kernel launch and top source lines."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Warp Cycles Per Issued Instruction", "Block Size", "Grid Size",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Compute (SM) Throughput"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, ni, ui, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value"), h.index("ID")
    res = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        if r[ni] in KEYS:
            res.setdefault((r[idi], r[ki][:60]), {})[r[ni]] = f"{r[vi]} {r[ui]}"
    return res


def raw(rep, pattern):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    cols = [i for i, c in enumerate(h) if any(p in c for p in pattern)]
    return [(h[i], rows[1][i], [r[i] for r in rows[2:]]) for i in cols]


def top_lines(rep, k=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, hdr, acc = None, None, []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1]
            continue
        if len(r) > 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) > 5 and r[0].isdigit():
            try:
                acc.append((int(r[4]), cur.split("/")[-1], int(r[0]), r[1][:100]))
            except ValueError:
                pass
    tot = sum(a[0] for a in acc) or 1
    acc.sort(reverse=True)
    return [f"{a[0]:8d} {100 * a[0] / tot:5.1f}% {a[1]}:{a[2]}  {a[3]}" for a in acc[:k]]


if __name__ == "__main__":
    rep = sys.argv[1]
    for key, m in details(rep).items():
        print(key)
        for kk in KEYS:
            if kk in m:
                print(f"   {kk:40s} {m[kk]}")
    if len(sys.argv) > 2:
        print("\n".join(top_lines(rep, int(sys.argv[2]))))
    for name, unit, vals in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum"]):
        if name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            print(name, unit, vals)
    print("pipe utilisation (% of peak, active cycles):")
    for name, unit, vals in raw(rep, ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                                      "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                                      "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                                      "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                                      "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]):
        print("  ", name, vals)
    print("warp stall samples:")
    st = [(name.replace("smsp__pcsamp_warps_issue_stalled_", ""), vals)
          for name, unit, vals in raw(rep, ["smsp__pcsamp_warps_issue_stalled_"]) if not name.endswith("not_issued")]
    tot = [sum(float(v[i] or 0) for _, v in st) or 1.0 for i in range(len(st[0][1]))] if st else []
    for name, vals in sorted(st, key=lambda x: -float(x[1][0] or 0))[:10]:
        print(f"   {name:28s}", " ".join(f"{100 * float(v or 0) / t:5.1f}%" for v, t in zip(vals, tot)))
