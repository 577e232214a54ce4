"""Summarise ncu output for profiles/ (run here on the .ncu-rep / CSV that a
gpurun call brought back).

  python tools/ncu_summary.py full  <rep.ncu-rep>  > profiles/<round>_<cfg>_full.md
  python tools/ncu_summary.py launches <launches.csv> > profiles/<round>_launches.md
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "time", 1.0),
    ("dram__bytes_read.sum", "dram rd", 1.0),
    ("dram__bytes_write.sum", "dram wr", 1.0),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %peak", 1.0),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %peak", 1.0),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %", 1.0),
    ("launch__registers_per_thread", "regs", 1.0),
    ("launch__grid_size", "grid", 1.0),
    ("launch__block_size", "block", 1.0),
    ("smsp__inst_executed.sum", "warp instr", 1.0),
]
STALLS = "smsp__average_warps_issue_stalled_"
STALL_SUFFIX = "_per_issue_active.ratio"


def _raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def full(rep):
    hdr, units, rows = _raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full summary: `{rep.split('/')[-1]}`\n")
    print("Captured with `ncu --set full --clock-control none --import-source on` (one process, "
          "cold caches, kernels serialised; times are NOT bench values).\n")
    head = ["kernel"] + [m[1] for m in FULL_METRICS] + ["top stalls (cycles/issue)"]
    print("| " + " | ".join(head) + " |")
    print("|" + "---|" * len(head))
    for r in rows:
        name = r[col["Kernel Name"]].split("(")[0]
        cells = [name]
        for m, _, _ in FULL_METRICS:
            if m not in col:
                cells.append("-")
                continue
            u = units[col[m]]
            v = r[col[m]].replace(",", "")
            cells.append(f"{v} {u}".strip())
        st = []
        for h, i in col.items():
            if h.startswith(STALLS) and h.endswith(STALL_SUFFIX):
                try:
                    st.append((float(r[i].replace(",", "")), h[len(STALLS):-len(STALL_SUFFIX)]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        cells.append(", ".join(f"{n} {v:.1f}" for v, n in st[:4]))
        print("| " + " | ".join(cells) + " |")


def launches(path):
    txt = open(path).read()
    lines = txt[txt.index('"ID"'):].splitlines()
    rows = list(csv.DictReader(lines))
    tot = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3,
                 "nsecond": 1e-3}.get(r.get("Metric Unit", "us"), 1.0)
        c, s = tot.get(k, (0, 0.0))
        tot[k] = (c + 1, s + v * scale)
    allt = sum(s for _, s in tot.values())
    print(f"# ncu launch list: `{path.split('/')[-1]}`\n")
    print("`ncu --metrics gpu__time_duration.sum --clock-control none` over the bench command; "
          "per-launch times are cold-cache and serialised, so compare SHARES, not absolutes.\n")
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---|---|---|---|")
    for k, (c, s) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {c} | {s:.1f} | {s / c:.1f} | {100 * s / allt:.1f}% |")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
