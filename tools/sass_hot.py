"""Summarise an ncu --page source --print-source sass CSV: instructions executed
per SASS line, average active threads, warp-stall samples.
Usage: python tools/sass_hot.py file.csv [min_exec]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc = h.index("Address"), h.index("Source")
iex, ith = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
ist = h.index("Warp Stall Sampling (All Samples)")
recs = []
for r in rows[2:]:
    if len(r) <= iex:
        continue
    try:
        recs.append((r[ia], r[isrc].strip(), int(r[iex] or 0), int(r[ith] or 0), int(r[ist] or 0)))
    except ValueError:
        pass
tot = sum(x[2] for x in recs); tst = sum(x[4] for x in recs)
print(f"total warp-instr {tot:,}  stall samples {tst:,}")
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for i, (a, s, ex, th, st) in enumerate(recs):
    if ex >= lo:
        print(f"{i:5d} {ex:12,d} {th/ex if ex else 0:5.1f} {st:7d}  {s}")
