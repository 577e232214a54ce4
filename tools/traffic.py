"""profiles/traffic.json from ncu --set full captures: DRAM bytes (read +
write) per build of each stage, summed over the stage's kernels.

  python tools/traffic.py C4=gpurun_out/r1b/full_sort_C4.ncu-rep,gpurun_out/r1b/full_emit_C4.ncu-rep ...
"""
import csv
import io
import json
import os
import subprocess
import sys

STAGE = {"k_hist": "plan", "k_plan": "plan", "k_hist_hi": "plan", "k_chunk_scan": "plan", "k_pass": "sort",
         "k_tma_pass": "sort", "k_pass_bytes": "sort", "k_set_row_hi": "sort", "k_vs": "sort",
         "k_tile_prep": "emit", "k_tile_heads": "emit", "k_emit": "emit", "k_emit_rows": "emit", "k_table": "table"}


def kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "").strip()
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[col[m]].replace(",", "")) * scale.get(units[col[m]], 1)
        yield name, b


def main():
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for arg in sys.argv[1:]:
        cfg, _, reps = arg.partition("=")
        per = {}
        for rep in reps.split(","):
            for name, b in kernels(rep):
                st = STAGE.get(name.split("::")[-1])
                if st:
                    per[st] = per.get(st, 0.0) + b
        data[cfg] = {k: int(v) for k, v in per.items()}
        data[cfg]["source"] = "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum, one build: " + reps
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
