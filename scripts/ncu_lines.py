"""Developer tool: per-source-line instruction and stall-sample totals from
`ncu --page source --csv --print-source cuda,sass` output.

    python scripts/ncu_lines.py SRC.csv [min_pct]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
minp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
hdr = next(r for r in rows if r and r[0] == "Line No")
ix = {k: i for i, k in enumerate(hdr)}
cur = None
agg = {}
order = []
seen = set()
fname = ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        cur = (fname, int(r[0]), r[1].strip()[:90])
        continue
    if len(r) < 5 or not r[2].startswith("0x") or r[2] in seen:
        continue
    seen.add(r[2])
    def g(k):
        try:
            return float(r[ix[k]] or 0)
        except (KeyError, ValueError):
            return 0.0
    a = agg.setdefault(cur, [0.0, 0.0, {}])
    if cur not in order:
        order.append(cur)
    a[0] += g("Warp Stall Sampling (All Samples)")
    a[1] += g("Instructions Executed")
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            a[2][k] = a[2].get(k, 0.0) + g(k)
ts = sum(v[0] for v in agg.values())
ti = sum(v[1] for v in agg.values())
print(f"samples {ts:.0f} warp-instructions {ti:.3e}")
for key in sorted(order, key=lambda k: (k[0], k[1])):
    s, n, st = agg[key]
    if 100 * s / ts < minp and 100 * n / ti < minp:
        continue
    top = sorted(st.items(), key=lambda x: -x[1])[:3]
    tops = " ".join(f"{k[6:]}:{100 * v / max(s, 1):.0f}%" for k, v in top)
    print(f"{key[0][:14]:14s}{key[1]:5d} {100 * s / ts:5.1f}% {100 * n / ti:5.1f}%  "
          f"{key[2][:58]:58s} {tops}")
