"""Summarise an ncu report (--set full) or an ncu launch-list CSV into markdown for profiles/.

    python tools/ncu_summary.py report.ncu-rep        # one kernel: SOL, memory, stalls
    python tools/ncu_summary.py launches.csv          # per-kernel time shares of a run
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors (from L1/TEX)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (achieved occupancy)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per warp instruction"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (v, u) for h, u, v in zip(hdr, units, r)} for r in rows[2:]]


def summarize_rep(rep):
    for rec in raw(rep):
        name = rec.get("Kernel Name", ("?", ""))[0]
        print(f"### `{name[:90]}`\n")
        print("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in rec:
                v, u = rec[k]
                print(f"| {label} (`{k}`) | {v} {u} |")
        stalls = []
        for k, (v, u) in rec.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        if stalls:
            stalls.sort(reverse=True)
            print("\nTop stall reasons (warps stalled per issued instruction): " +
                  ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))
        print()


def summarize_csv(path):
    rows = list(csv.reader(open(path)))
    i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[i]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
             "second": 1e3}
    for r in rows[i + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].strip()[:70]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {c} | {ms:.3f} | {100 * ms / tot:.2f} % |")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        (summarize_csv if p.endswith(".csv") else summarize_rep)(p)
