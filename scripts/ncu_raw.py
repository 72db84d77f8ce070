"""Selected raw metrics (columns matching any regex argument) of ncu raw CSVs:
python scripts/ncu_raw.py 'tensor|stall' gpurun_out/raw_<tag>.csv ..."""
import csv
import re
import sys

pat = re.compile(sys.argv[1])
for path in sys.argv[2:]:
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    print("==", path)
    for r in rows[2:]:
        for h, u, v in zip(hdr, units, r):
            if pat.search(h) and v not in ("", "0", "0.00", "n/a"):
                print(f"   {h[:90]:90s} {v:>16s} {u}")
