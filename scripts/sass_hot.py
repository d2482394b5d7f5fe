"""Summarise an `ncu --page source --csv` dump: hottest SASS lines by stall samples and opcode mix."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Source" in r and "# Samples" in r)
hdr = rows[h]
ia, ie, isamp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("# Samples")
data = []
for r in rows[h + 1:]:
    try:
        data.append((r[ia].strip(), int(r[ie]), int(r[isamp])))
    except (ValueError, IndexError):
        pass
tot = sum(d[1] for d in data) or 1
ts = sum(d[2] for d in data) or 1
print("total warp instr", tot, "samples", ts, "sass lines", len(data))
for src, n, sm in sorted(data, key=lambda d: -d[2])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{100 * sm / ts:5.1f}% samp {100 * n / tot:5.1f}% inst  {src[:100]}")
hist = collections.Counter()
for src, n, sm in data:
    parts = src.split()
    op = parts[1] if parts and parts[0].startswith("@") else (parts[0] if parts else "?")
    hist[op.split(".")[0]] += n
print([(k, round(100 * v / tot, 1)) for k, v in hist.most_common(20)])
