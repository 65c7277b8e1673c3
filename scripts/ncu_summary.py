"""Summarise ncu captures into profiles/ (developer tool; needs `ncu` on PATH).

    python scripts/ncu_summary.py full  REP.ncu-rep[#i] OUT.txt # --set full capture (i-th kernel)
    python scripts/ncu_summary.py launches LAUNCHES.csv OUT.txt # gpu__time_duration list
    python scripts/ncu_summary.py traffic OUT.json NAME=REP.ncu-rep[#i] ... --note "..." [--workload W]
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
]


def raw(rep):
    """(header, units, values) of kernel i of REP#i (default 0)."""
    idx = 0
    if "#" in rep:
        rep, i = rep.rsplit("#", 1)
        idx = int(i)
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2 + idx]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * scale.get(unit, 1)


def full(rep, out):
    h, u, v = raw(rep)
    lines = [f"# ncu --set full summary of {rep.split('/')[-1]}"]
    lines.append(f"kernel: {v[h.index('Kernel Name')][:160]}")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            lines.append(f"{k} = {v[i]} {u[i]}")
    lines.append("# warp stall reasons (per issued instruction)")
    for k, x, un in zip(h, v, u):
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                if float(x) >= 0.05:
                    lines.append(f"{k.replace('smsp__average_warps_issue_stalled_', 'stall_')} = {x}")
            except ValueError:
                pass
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        k = r[iN].split("(")[0].replace("void ", "")
        tot[k] += float(r[iV].replace(",", "")) * scale.get(r[iU], 1e-6)
        cnt[k] += 1
    T = sum(tot.values())
    lines = [f"# launch list {path.split('/')[-1]}: {sum(cnt.values())} launches, {T:.2f} ms "
             "(cold-cache, serialised: compare shares, not absolutes)",
             f"{'kernel':48s} {'n':>5s} {'ms':>9s} {'share':>7s}"]
    for k, ms in tot.most_common():
        lines.append(f"{k[:48]:48s} {cnt[k]:5d} {ms:9.3f} {ms / T * 100:6.1f}%")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def traffic(out, pairs, note, workload=None):
    """Writes OUT as {"workloads": {WORKLOAD: {"source", "kernels"}}}, merging
    into an existing file (bench.py reads the entry of the workload it runs)."""
    d = {"source": note, "kernels": {}}
    for p in pairs:
        name, rep = p.split("=", 1)
        h, u, v = raw(rep)
        rd = to_bytes(v[h.index("dram__bytes_read.sum")], u[h.index("dram__bytes_read.sum")])
        wr = to_bytes(v[h.index("dram__bytes_write.sum")], u[h.index("dram__bytes_write.sum")])
        t = float(v[h.index("gpu__time_duration.sum")].replace(",", ""))
        tu = u[h.index("gpu__time_duration.sum")]
        d["kernels"][name] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                              "duration": f"{t} {tu}", "report": rep.split("/")[-1]}
    if workload:
        try:
            allw = json.load(open(out))
            if "workloads" not in allw:
                allw = {"workloads": {}}
        except Exception:
            allw = {"workloads": {}}
        allw["workloads"][workload] = d
        d = allw
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        full(sys.argv[2], sys.argv[3])
    elif mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        args = sys.argv[3:]
        note = ""
        if "--note" in args:
            i = args.index("--note")
            note = args[i + 1]
            args = args[:i] + args[i + 2:]
        wl = None
        if "--workload" in args:
            i = args.index("--workload")
            wl = args[i + 1]
            args = args[:i] + args[i + 2:]
        traffic(sys.argv[2], args, note, wl)
