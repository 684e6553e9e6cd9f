"""Aggregate an ncu `--page source --print-source sass --csv` dump: warp instructions and
stall samples per opcode, and the hottest address ranges (dev tool)."""
import csv, sys, collections

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = rows[2:]
tot_i = tot_s = 0
by_op = collections.Counter(); st_op = collections.Counter()
recs = []
for r in body:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    base = op.split(".")[0]
    ni = int(r[ix["Instructions Executed"]] or 0)
    ns = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot_i += ni; tot_s += ns
    by_op[base] += ni; st_op[base] += ns
    recs.append((r[ix["Address"]], src, ni, ns))
print(f"total warp instructions {tot_i/1e6:.1f} M, stall samples {tot_s}")
for op, n in by_op.most_common(30):
    print(f"  {op:12s} {n/1e6:8.2f} M  {100*n/tot_i:5.1f} %   stall {100*st_op[op]/max(tot_s,1):5.1f} %")
if len(sys.argv) > 2:
    win = int(sys.argv[2])
    # sliding windows of `win` instructions by instruction count
    best = []
    for i in range(0, len(recs), win):
        seg = recs[i:i + win]
        best.append((sum(s[2] for s in seg), sum(s[3] for s in seg), seg[0][0], seg[-1][0]))
    for ni, ns, a0, a1 in sorted(best, reverse=True)[:15]:
        print(f"  {a0}-{a1}: {ni/1e6:7.2f} M instr  {ns} samples")
