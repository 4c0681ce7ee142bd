"""Per-region stall breakdown of an ncu --page source --csv --print-source sass dump."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
step = int(sys.argv[2]) if len(sys.argv) > 2 else 50
h = rows[1]; data = rows[2:]
si = h.index('Warp Stall Sampling (All Samples)'); ei = h.index('Instructions Executed')
reasons = [c for c in h if c.startswith('stall_') and '(Not' not in c]
ri = {c: h.index(c) for c in reasons}
num = lambda v: float(v) if v not in ('', '-') else 0.0
tot = sum(num(r[si]) for r in data); totx = sum(num(r[ei]) for r in data)
print('samples', tot, 'instr', len(data), 'exec', totx)
for k in range(0, len(data), step):
    ch = data[k:k + step]
    ss = sum(num(r[si]) for r in ch)
    if ss < tot * 0.01: continue
    sx = sum(num(r[ei]) for r in ch)
    st = collections.Counter({c: sum(num(r[ri[c]]) for r in ch) for c in reasons})
    ops = collections.Counter(r[1].split()[0] if not r[1].split()[0].startswith('@') else r[1].split()[1] for r in ch)
    print(f"{k:5d} samp {ss/tot*100:4.1f}% exec {sx/totx*100:4.1f}% | " +
          ' '.join(f"{c[6:]}:{v/ss*100:.0f}" for c, v in st.most_common(3)) + " | " +
          ' '.join(f"{o}:{n}" for o, n in ops.most_common(4)))
