"""Instructions executed and stall samples of an ncu source capture grouped
into line ranges (phases). Usage: ncu_phases.py REP file.cu name:first-last ..."""
import csv, io, subprocess, sys
rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    nm, r = a.split(":"); lo, hi = r.split("-"); ranges.append((nm, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr = None, None
tot = {nm: [0, 0] for nm, _, _ in ranges}; tot["other"] = [0, 0]
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r; continue
    if hdr and len(r) > 6 and r[0].isdigit():
        try:
            ie = int(r[hdr.index("Instructions Executed")]); smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        ln = int(r[0]); key = "other"
        if cur == fname:
            for nm, lo, hi in ranges:
                if lo <= ln <= hi: key = nm
        tot[key][0] += ie; tot[key][1] += smp
TI = sum(v[0] for v in tot.values()) or 1; TS = sum(v[1] for v in tot.values()) or 1
print(f"total warp-instructions {TI}, samples {TS}")
for k, v in tot.items():
    print(f"{k:10s} inst {100*v[0]/TI:5.1f}%  stall-samples {100*v[1]/TS:5.1f}%")
