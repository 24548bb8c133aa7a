import re,sys
rows=[]
for l in open(sys.argv[1]):
    m=re.match(r'\s*(\d+)\s+([\d.]+)%\s+smp\s+([\d.]+)%\s+(\S+)\s+(.*)',l)
    if m: rows.append((float(m.group(3)),float(m.group(2)),m.group(4),m.group(5)[:90]))
rows.sort(reverse=True)
for r in rows[:int(sys.argv[2])]: print(f"smp {r[0]:5.1f}% inst {r[1]:5.1f}%  {r[2]}  {r[3]}")
