"""Warp-stall samples by SASS instruction from `ncu -i <rep> --page source --csv --print-source sass`
(a capture taken with --import-source on): by opcode and the top instructions, as markdown.
usage: ncu -i rep --page source --csv --print-source sass > src.csv; python tools/sass_stalls.py src.csv"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
ci = {k: hdr.index(k) for k in ("Source", "Warp Stall Sampling (All Samples)", "Avg. Threads Executed")}
recs = []
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr):
        continue
    try:
        n = int(r[ci["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    recs.append((r[ci["Source"]].strip(), n, r[ci["Avg. Threads Executed"]]))
tot = sum(n for _, n, _ in recs) or 1
ops = Counter()
for src, n, _ in recs:
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    ops[op.split(".")[0]] += n
print(f"{tot} stall samples in total\n\n## By opcode\n\n| opcode | share |\n|---|---|")
for op, n in ops.most_common(12):
    print(f"| `{op}` | {100 * n / tot:.1f}% |")
print("\n## Top 20 instructions\n\n| SASS | share | avg threads executed |\n|---|---|---|")
for src, n, th in sorted(recs, key=lambda x: -x[1])[:20]:
    print(f"| `{src}` | {100 * n / tot:.1f}% | {th} |")
