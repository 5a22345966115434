"""Per-launch DRAM traffic of each kernel class from an `ncu --set full` report -> profiles/ncu_traffic.json
(bench.py reports it as roofline.traffic).   python tools/ncu_traffic.py REPORT.ncu-rep OUT.json [workload]"""
import csv
import io
import json
import subprocess
import sys

CLASSES = [("k_rhs_r2c", "rhs_r2c"), ("k_rhs", "rhs"), ("k_wb", "wb"), ("k_rows_r2c", "rows_r2c"), ("k_cols_solve", "cols_solve"), ("k_cols_tri", "cols_solve"),
           ("k_rows_c2r", "rows_c2r"), ("k_aos_vert", "aos_vert"), ("k_aos_horiz", "aos_horiz")]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    workload = sys.argv[3] if len(sys.argv) > 3 else "c3"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    names = {}
    for d in data:
        name = d[col["Kernel Name"]]
        cls = next((c for p, c in CLASSES if p in name), None)
        if cls is None:
            continue
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d[col[m]].replace(",", "")) * scale[units[col[m]]]
        per.setdefault(cls, []).append(tot)
        names[cls] = name.split("(")[0]
    res = {"workload": workload,
           "source": f"{rep}: ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over "
                     f"captured launches)",
           "kernels": names,
           "per_launch_bytes": {k: sum(v) / len(v) for k, v in per.items()}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
