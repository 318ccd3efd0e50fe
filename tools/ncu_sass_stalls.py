"""Summarise an ncu --page source --csv --print-source sass dump: stall
samples by opcode and by stall reason, the hottest sites, and per-region
totals (contiguous address ranges split at BAR.SYNC / EXIT)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    samples = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = {c: int(r[ix[c]] or 0) for c in stall_cols}
    ex = int(r[ix["Instructions Executed"]] or 0)
    data.append((r[ix["Address"]], src, op.split(".")[0], samples, st, ex))
tot = sum(d[3] for d in data)
print("total samples", tot)
by_op = defaultdict(int)
by_reason = defaultdict(int)
by_op_reason = defaultdict(lambda: defaultdict(int))
for a, s, op, n, st, ex in data:
    by_op[op] += n
    for c, v in st.items():
        by_reason[c] += v
        by_op_reason[op][c] += v
print("\nby opcode (% samples):")
for op, n in sorted(by_op.items(), key=lambda x: -x[1])[:15]:
    top = sorted(by_op_reason[op].items(), key=lambda x: -x[1])[:4]
    print(f"  {op:10s} {100*n/tot:5.1f}%  ", ", ".join(f"{c[6:]} {100*v/tot:.1f}" for c, v in top))
print("\nby reason (% samples):")
for c, v in sorted(by_reason.items(), key=lambda x: -x[1])[:12]:
    print(f"  {c:24s} {100*v/tot:5.1f}%")
print("\nhottest sites:")
for a, s, op, n, st, ex in sorted(data, key=lambda x: -x[3])[:25]:
    top = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"  {a[-5:]} {100*n/tot:5.2f}% ex={ex:9d} {s[:60]:60s} ", ", ".join(f"{c[6:]} {v}" for c, v in top))
# regions between barriers
print("\nregions (split at BAR.SYNC):")
reg, cur = [], []
for d in data:
    cur.append(d)
    if d[2] in ("BAR", "EXIT"):
        reg.append(cur)
        cur = []
reg.append(cur)
for i, rg in enumerate(reg):
    n = sum(d[3] for d in rg)
    if n < 0.01 * tot:
        continue
    ex = sum(d[5] for d in rg)
    dfma = sum(d[5] for d in rg if d[2] in ("DFMA", "DADD", "DMUL"))
    print(f"  region {i}: {rg[0][0][-5:]}..{rg[-1][0][-5:]} {len(rg)} instrs, {100*n/tot:.1f}% samples,"
          f" exec {ex}, fp64 exec {dfma}")
if len(sys.argv) > 2:
    lo, hi = (int(x, 16) for x in sys.argv[2].split(":"))
    sub = [d for d in data if lo <= int(d[0], 16) % (1 << 20) <= hi]
    n = sum(d[3] for d in sub)
    rs = defaultdict(int)
    ops = defaultdict(lambda: [0, 0])
    for a, s, op, k, st, ex in sub:
        for c, v in st.items():
            rs[c] += v
        ops[op][0] += ex
        ops[op][1] += k
    print(f"\nrange {sys.argv[2]}: {len(sub)} instrs, {n} samples")
    for c, v in sorted(rs.items(), key=lambda x: -x[1])[:10]:
        print(f"  {c:24s} {100*v/n:5.1f}%")
    print("  executed by opcode:", ", ".join(f"{o} {e}" for o, (e, k) in sorted(ops.items(), key=lambda x: -x[1][0])[:14]))
