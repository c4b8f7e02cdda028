"""DRAM traffic of one query step from an ncu capture of bench.py's own command (its own
fixture), for bench.py's `roofline.traffic` (profiles/r02_traffic.json).

  python tools/traffic_from_ncu.py REPORT.ncu-rep --config 3 --kernels k_bin_tma,k_query_regions,k_unbin_tma \
      --cmd "the profiled command" [--out profiles/r02_traffic.json]

Sums dram__bytes_read.sum + dram__bytes_write.sum over the first launch of each named kernel
(one step of the path) and records the per-kernel figures beside the total.
"""
import argparse
import csv
import io
import json
import os
import subprocess

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--kernels", required=True)
    ap.add_argument("--cmd", required=True)
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "profiles", "r02_traffic.json"))
    a = ap.parse_args()
    if a.report.endswith(".csv"):  # `ncu -i X.ncu-rep --page raw --csv` already run on the GPU box
        with open(a.report) as f:
            raw = f.read()
    else:
        raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {m: hdr.index(m) for m in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                     "gpu__time_duration.sum")}
    want = a.kernels.split(",")
    per = {}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        k = next((w for w in want if w in name), None)
        if not k or k in per:
            continue
        rd = float(r[col["dram__bytes_read.sum"]]) * UNITS[units[col["dram__bytes_read.sum"]]]
        wr = float(r[col["dram__bytes_write.sum"]]) * UNITS[units[col["dram__bytes_write.sum"]]]
        wf_col = "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg"
        wf = float(r[hdr.index(wf_col)]) if wf_col in hdr and r[hdr.index(wf_col)] else None
        per[k] = {"dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
                  "lsu_wavefronts_per_sm": wf,  # L1 data-pipe wavefronts, average per SM
                  "ncu_ms": float(r[col["gpu__time_duration.sum"]]) *
                  (1e-3 if units[col["gpu__time_duration.sum"]] == "usecond" else 1.0)}
    missing = [k for k in want if k not in per]
    if missing:
        raise SystemExit(f"kernels not in the report: {missing}")
    d = {}
    if os.path.exists(a.out):
        with open(a.out) as f:
            d = json.load(f)
    d[f"config{a.config}"] = {
        "dram_bytes_per_step": sum(v["dram_read_bytes"] + v["dram_write_bytes"] for v in per.values()),
        "kernels": per,
        "source": f"ncu --set full capture ({os.path.basename(a.report)}) of `{a.cmd}`: first "
                  f"launch of each of {', '.join(want)} on the bench's own fixture; "
                  f"dram__bytes_read.sum + dram__bytes_write.sum",
    }
    with open(a.out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(d[f"config{a.config}"], indent=1))


if __name__ == "__main__":
    main()
