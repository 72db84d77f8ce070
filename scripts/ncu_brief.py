"""Compact view of an ncu report's details page: python scripts/ncu_brief.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ki, si, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
seen = None
for r in rows[1:]:
    if len(r) != len(hdr):
        continue
    if r[ki] != seen:
        seen = r[ki]
        print("==", r[ki][:80])
    print(f"  {r[si][:28]:28s} {r[mi][:40]:40s} {r[vi]:>14s} {r[ui]}")
