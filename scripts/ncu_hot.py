"""Hot SASS lines of one kernel from `ncu -i rep --page source --csv --kernel-name regex:NAME` output (stdin or file)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.006
h = rows[1]
si, ii, src = h.index("# Samples"), h.index("Instructions Executed"), h.index("Source")
recs = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) > max(si, ii) and r[si].isdigit():
        recs.append(r)
tot_s = sum(int(r[si]) for r in recs); tot_i = sum(int(r[ii]) for r in recs)
print("total samples", tot_s, "instr", tot_i, "SASS lines", len(recs))
for k, r in enumerate(recs):
    s = int(r[si])
    if s > thr * tot_s:
        print(f"{k:5d} {100*s/tot_s:5.1f}% smp  {int(r[ii])/1e6:7.2f}M  {r[src].strip()[:100]}")
