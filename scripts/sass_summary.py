"""Per-kernel SASS instruction-class counts of the built library (static
counts from cuobjdump): the tcgen05 / TMA evidence for each tensor-core
kernel. Developer tool (CPU only).

    python scripts/sass_summary.py [OBJ ...] > profiles/r02_sass_counts.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLASSES = [
    ("UTCHMMA", "tcgen05.mma (kind::f16)"),
    ("UTCQMMA", "tcgen05.mma (other kinds)"),
    ("UTCBAR", "tcgen05.commit -> mbarrier"),
    ("LDTM", "tcgen05.ld (TMEM -> registers)"),
    ("STTM", "tcgen05.st (registers -> TMEM)"),
    ("UTMALDG", "TMA tensor load (cp.async.bulk.tensor)"),
    ("UBLKCP", "bulk copy (cp.async.bulk)"),
    ("LDGSTS", "cp.async (global -> shared)"),
    ("SYNCS", "mbarrier ops"),
    ("USETMAXREG", "setmaxnreg"),
    ("MUFU.EX2", "ex2"),
    ("FFMA2", "packed fp32 FMA"),
    ("HMMA", "legacy mma.sync"),
]


def main():
    objs = sys.argv[1:] or [os.path.join(ROOT, "paper_2212_11296_b200", "_lib", f)
                            for f in ("engine.cu.o", "grad.cu.o")]
    print("# static SASS instruction counts per kernel (cuobjdump -sass; sm_100a)")
    for obj in objs:
        out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        counts = collections.OrderedDict()
        cur = None
        for ln in out.splitlines():
            m = re.match(r"\s+Function : (\S+)", ln)
            if m:
                cur = m.group(1)
                counts[cur] = collections.Counter()
                continue
            if cur is None:
                continue
            m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
            if not m:
                continue
            op = m.group(2)
            counts[cur]["total"] += 1
            for key, _ in CLASSES:
                if op.startswith(key):
                    counts[cur][key] += 1
        print(f"\n## {os.path.basename(obj)}")
        print("kernel".ljust(60) + "".join(k.split(".")[0][:8].rjust(9) for k, _ in CLASSES) + "    total")
        for fn, c in counts.items():
            if not any(c[k] for k, _ in CLASSES[:8]):
                continue
            name = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
            name = re.sub(r"\(.*", "", name)[:58]
            print(name.ljust(60) + "".join(str(c[k]).rjust(9) for k, _ in CLASSES) +
                  str(c["total"]).rjust(9))
    print("\nclasses: " + "; ".join(f"{k} = {v}" for k, v in CLASSES))


if __name__ == "__main__":
    main()
