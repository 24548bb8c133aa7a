"""profiles/ summaries from this round's ncu captures:
  * r02_launches_<cfg>.txt: per-kernel time / launches / DRAM bytes of one
    steady-state BFM iteration (ncu launch list, --profile-from-start off);
  * dram_bytes.json: DRAM bytes (read + write) per operator call, keyed
    "<op>@<grid>", for bench.py's roofline `traffic` fields.
Usage: python tools/dram_table.py gpurun_out/r02f_launches_c3.csv gpurun_out/r02f_launches_c4.csv"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = {  # kernel -> operator of bench.py's rooflines
    "ct_dy_kernel": "ctransform", "ct_pass_kernel": "ctransform",
    "ct_transpose_f64": "ctransform", "ct_transpose_state": "ctransform",
    "pois_fft_kernel": "poisson", "pois_naive_kernel": "poisson",
    "red_partial_kernel": "reductions", "red_final_kernel": "reductions", "axpy_dev_kernel": "reductions",
    "ctl_decide_kernel": "reductions",
}
CALLS = {"ctransform": 4, "pushforward": 2, "poisson": 2, "reductions": 1}  # per iteration


def parse(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    data = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1.0)
        else:
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        data[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].split("::")[-1].split("<")[0]
    return data, names


def main():
    table = {}
    try:
        table = json.load(open(os.path.join(ROOT, "profiles", "dram_bytes.json")))
    except Exception:
        pass
    for path in sys.argv[1:]:
        cfg = "c3" if "c3" in os.path.basename(path) else "c4"
        grid = "4096x4096" if cfg == "c3" else "384x384x384"
        data, names = parse(path)
        per_kernel = collections.defaultdict(lambda: [0.0, 0, 0.0])
        per_op = collections.defaultdict(float)
        for i, d in data.items():
            k = names[i]
            b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            t = per_kernel[k]
            t[0] += d.get("gpu__time_duration.sum", 0)
            t[1] += 1
            t[2] += b
            per_op[OPS.get(k, "pushforward" if k.startswith(("pf_", "rs_", "os_")) else "other")] += b
        T = sum(v[0] for v in per_kernel.values())
        lines = [f"# one steady-state {cfg.upper()} iteration ({grid}) after 8 warm-up iterations, "
                 f"eager launches (ncu --profile-from-start off, --clock-control none; serialised, cold-cache "
                 f"per-launch times: shares, not absolute step time)",
                 f"# total {T / 1e3:.2f} ms over {sum(v[1] for v in per_kernel.values())} launches",
                 "#   ms   launches  share  DRAM MB/launch  GB/s   kernel"]
        for k, v in sorted(per_kernel.items(), key=lambda x: -x[1][0]):
            lines.append(f"{v[0] / 1e3:8.3f} {v[1]:5d} {100 * v[0] / T:6.1f}% {v[2] / 1e6 / v[1]:10.1f} "
                         f"{v[2] / (v[0] * 1e-6) / 1e9 if v[0] else 0:7.0f}  {k}")
        out = os.path.join(ROOT, "profiles", f"r02_launches_{cfg}.txt")
        open(out, "w").write("\n".join(lines) + "\n")
        print(open(out).read())
        for op, b in per_op.items():
            if op in CALLS:
                table[f"{op}@{grid}"] = b / CALLS[op]
    table["_note"] = ("DRAM bytes (ncu dram__bytes_read.sum + dram__bytes_write.sum) per operator call inside one "
                      "steady-state iteration (reductions: per iteration), from profiles/r02_launches_<cfg>.txt "
                      "(tools/dram_table.py); bench.py's roofline `traffic`")
    json.dump(table, open(os.path.join(ROOT, "profiles", "dram_bytes.json"), "w"), indent=1, sort_keys=True)
    print(json.dumps(table, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
