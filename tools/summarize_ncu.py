"""Summarise ncu raw-page CSV exports (tools/profile_all.sh) into a markdown
table: duration, DRAM bytes vs algorithmic bytes, achieved GB/s, occupancy,
issue activity, top stall reasons.  usage: python tools/summarize_ncu.py DIR > out.md"""
import csv
import glob
import os
import sys

ALG = {  # algorithmic bytes per launch of tools/profile_step.py workloads
    "c2": 1.6e9, "c2ro": 1.2e9, "axpy": (1 << 30) * 12, "c3d0": (1 << 30) * 8 + 32768 * 8,
    "c3d1": (1 << 30) * 8 + 32768 * 8, "c4u": (1 << 28) * 12, "c4s": (1 << 28) * 24,
    "dot": (1 << 30) * 8, "norm2": (1 << 30) * 4,
}
DESC = {
    "c2": "exp(A%B)+3C, Z stored + accu, 1e8 f32", "c2ro": "accu(exp(A%B)+3C), 1e8 f32",
    "axpy": "y=2.5x+y + accu, 2^30 f32", "c3d0": "sum(X,0), 32768^2 f64",
    "c3d1": "sum(X,1), 32768^2 f64", "c4u": "minmax(X%Y+7Z), 2^28 u32",
    "c4s": "minmax(X%Y+7Z), 2^28 s64", "dot": "dot(x,y), 2^30 f32", "norm2": "norm2(x), 2^30 f32",
}


def scale(v, u):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3,
         "nsecond": 1e-9, "second": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}
    return float(v) * f.get(u, 1)


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def main(d):
    print("| workload | kernel | time (us) | DRAM bytes | alg bytes | DRAM/alg | achieved GB/s | dram % peak | regs | warps active % | issue active % | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for p in sorted(glob.glob(os.path.join(d, "raw_*.csv"))):
        w = os.path.basename(p)[4:-4]
        try:
            m = load(p)
        except Exception:
            continue
        t = scale(*m["gpu__time_duration.sum"])
        db = scale(*m["dram__bytes_read.sum"]) + scale(*m["dram__bytes_write.sum"])
        alg = ALG.get(w, 0)
        st = sorted([(k, float(v[0] or 0)) for k, v in m.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")],
                    key=lambda x: -x[1])
        tot = sum(x[1] for x in st) or 1
        stalls = ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%"
                           for k, v in st[:3])
        name = m["Kernel Name"][0].split("(")[0].replace("void ", "")[:60]
        print(f"| {w}: {DESC.get(w, '')} | `{name}` | {t * 1e6:.1f} | {db:.4g} | {alg:.4g} | "
              f"{db / alg if alg else 0:.3f} | {alg / t / 1e9 if alg else 0:.0f} | "
              f"{float(m['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'][0]):.1f} | "
              f"{m['launch__registers_per_thread'][0]} | "
              f"{float(m['sm__warps_active.avg.pct_of_peak_sustained_active'][0]):.1f} | "
              f"{float(m['smsp__issue_active.avg.pct_of_peak_sustained_active'][0]):.1f} | {stalls} |")


if __name__ == "__main__":
    main(sys.argv[1])
