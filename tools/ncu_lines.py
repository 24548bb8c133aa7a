"""Per-source-line totals from an ncu report (--import-source): instructions
executed and warp-stall samples, aggregated over the SASS of each line."""
import csv, io, subprocess, sys
rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, acc = None, None, {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r; continue
    if hdr and len(r) > 6 and r[0].isdigit():
        try:
            ie = int(r[hdr.index("Instructions Executed")]) if "Instructions Executed" in hdr else 0
            smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        key = (cur, int(r[0]))
        a = acc.setdefault(key, [0, 0, r[1][:90]])
        a[0] += ie; a[1] += smp
tot_i = sum(v[0] for v in acc.values()) or 1
tot_s = sum(v[1] for v in acc.values()) or 1
print(f"total warp-instructions {tot_i}  samples {tot_s}")
for key, v in sorted(acc.items(), key=lambda kv: -kv[1][0])[:k]:
    print(f"{v[0]:10d} {100*v[0]/tot_i:5.1f}%  smp {100*v[1]/tot_s:5.1f}%  {key[0]}:{key[1]}  {v[2]}")
