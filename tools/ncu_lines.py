"""Per-source-line instruction and stall-sample shares of one kernel from an
ncu report (needs -lineinfo builds and --import-source on).
    python tools/ncu_lines.py <rep.ncu-rep> <function substring> [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep, fn = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = {}
    path, func, hdr, seen = None, None, None, set()
    take = False
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1]
            continue
        if r[0] == "Function Name":
            func = r[1]
            key = (path, func)
            take = fn in func and key not in seen  # first instance (launch) of each file section
            seen.add(key)
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if not take or not r[0]:
            continue
        try:
            ins = int(r[hdr["Instructions Executed"]] or 0)
            smp = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, KeyError, IndexError):
            continue
        k = (path.split("/")[-1], int(r[0]))
        a = agg.setdefault(k, [0, 0, r[1].strip()[:100]])
        a[0] += ins
        a[1] += smp
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"{fn}: {ti} warp instructions, {ts} stall samples")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * v[0] / ti:5.1f}% ins {100 * v[1] / ts:5.1f}% smp  {k[0]}:{k[1]}  {v[2]}")


if __name__ == "__main__":
    main()
