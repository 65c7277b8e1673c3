"""Developer tool: per-kernel DRAM traffic and achieved bandwidth from an
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
lts__t_bytes.sum --csv` launch list.

    python scripts/ncu_memk.py LAUNCHES.csv [peak_GBps]
"""
import collections
import csv
import sys

SC = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9,
      "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6553.0
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) >= 15 and r[0].isdigit()]
    per = collections.defaultdict(dict)
    for r in rows:
        name = r[4].split("(")[0]
        per[(name, r[0])][r[12]] = float(r[14].replace(",", "")) * SC.get(r[13], 1.0)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (k, _), d in per.items():
        a = agg[k]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a[3] += d.get("lts__t_bytes.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':34s} {'launches':>8s} {'ms':>8s} {'share':>6s} {'DRAM GB':>8s} "
          f"{'DRAM GB/s':>9s} {'% peak':>6s} {'L2 GB/s':>8s}")
    for k, (n, t, b, l2) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:34]:34s} {n:8d} {t * 1e3:8.3f} {t / tot * 100:5.1f}% {b / 1e9:8.3f} "
              f"{b / t / 1e9:9.0f} {b / t / 1e9 / peak * 100:6.1f} {l2 / t / 1e9:8.0f}")


if __name__ == "__main__":
    main()
