"""Summarise an ncu export: headline sections, busy pipes, top stalls and the
SASS instruction mix per element.

usage: python tools/ncu_mix.py PREFIX N_ELEMENTS
  reads PREFIX_details.csv, PREFIX_raw.csv, PREFIX_sass.csv (ncu -i ... --page
  details|raw|source --csv [--print-source sass]).
"""
import collections
import csv
import sys


def details(prefix):
    rows = list(csv.reader(open(prefix + "_details.csv")))
    h = rows[0]
    keep = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
            "Issue Slots Busy", "Executed Ipc Active", "Warp Cycles Per Issued Instruction",
            "Achieved Occupancy", "Registers Per Thread", "Executed Instructions")
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in keep:
            print(f"  {d['Metric Name']:40s} {d['Metric Value']:>14s} {d.get('Metric Unit', '')}")


def raw(prefix):
    rows = list(csv.reader(open(prefix + "_raw.csv")))
    h, v = rows[0], rows[2]
    pipes, stalls = [], []
    for k, x in zip(h, v):
        try:
            f = float(x.replace(",", ""))
        except ValueError:
            continue
        if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active"):
            pipes.append((f, k[len("sm__inst_executed_pipe_"):].split(".")[0]))
        if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio"):
            stalls.append((f, k[len("smsp__average_warp_latency_issue_stalled_"):].split(".")[0]))
    print("  pipes %:", ", ".join(f"{n} {p:.1f}" for p, n in sorted(pipes, reverse=True)[:8]))
    if stalls:
        print("  stalls :", ", ".join(f"{n} {p:.2f}" for p, n in sorted(stalls, reverse=True)[:6]))


def sass(prefix, n_elem):
    rows = list(csv.reader(open(prefix + "_sass.csv")))
    for i, r in enumerate(rows):
        if "Source" in r and "Instructions Executed" in r:
            h, start = r, i
            break
    si, ie = h.index("Source"), h.index("Instructions Executed")
    cnt = collections.Counter()
    for r in rows[start + 1:]:
        if len(r) <= ie:
            continue
        try:
            n = int(r[ie].replace(",", ""))
        except ValueError:
            continue
        toks = r[si].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        cnt[op.split(".")[0]] += n
    warps = n_elem / 32
    tot = sum(cnt.values())
    print(f"  warp-instructions per element-warp: {tot / warps:.1f}")
    print("  " + ", ".join(f"{k} {v / warps:.2f}" for k, v in cnt.most_common(24)))


if __name__ == "__main__":
    p, n = sys.argv[1], float(sys.argv[2])
    print(p)
    details(p)
    raw(p)
    sass(p, n)
