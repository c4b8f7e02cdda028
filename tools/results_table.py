"""Regenerates DESIGN.md §4's results table, the partition-pass summary, the config-3
speed-ups and README.md's results rows from the committed bench lines
(profiles/r01_bench_config*.json, profiles/r01_bench_reference_config3.json).

  python tools/results_table.py
"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(name):
    with open(os.path.join(ROOT, "profiles", name)) as f:
        return json.load(f)


def main():
    d = {c: load(f"r01_bench_config{c}.json") for c in (1, 2, 3, 4, 5)}
    r = load("r01_bench_reference_config3.json")
    d3, d5 = d[3], d[5]

    def row(c, label, extra=""):
        x = d[c]
        ms = f"{x['ms_per_step']:.3f}" if c == 1 else f"{x['ms_per_step']:.2f}"
        v = f"**{x['value']:.1f}**" if c == 3 else f"{x['value']:.1f}"
        e = f"**{x['e2e']['value']:.2f}**" if c == 3 else f"{x['e2e']['value']:.2f}"
        return (f"| {label} | {v} ({ms} ms) | {x['nonminimal']['value']:.1f} | {e} | "
                f"{x['cpu_baseline']['value']:.2f} | {x['roofline']['frac']:.2f}{extra} | "
                f"{x['gather_roofline']['frac']:.2f} |")

    table = "\n".join([
        row(3, "**3 (headline)** | 1e9 u64, shuffled; partitioned path (default layout)"),
        row(5, "5 | 1e9 k-mers, fused front end, partitioned path"),
        row(4, "4 | 3e8 strings, AES, shuffled"),
        row(2, "2 | 1e8 queries, 33 MB pilots", " (L2-resident)"),
        row(1, "1 | 1e7 u64, shuffled", " (L2-resident)"),
    ])
    p3, p5 = d3["partition_passes"], d5["partition_passes"]
    passes = (f"Per-pass rooflines of the partitioned path (bench.py `partition_passes`, live CUDA events):\n"
              f"config 3 bin {p3['bin']['ms']:.2f} ms ({p3['bin']['frac']:.2f} of HBM), query {p3['query']['ms']:.2f} ms\n"
              f"({p3['query']['frac']:.2f} of the L2 gather rate), unbin {p3['unbin']['ms']:.2f} ms ({p3['unbin']['frac']:.2f} of HBM);\n"
              f"config 5 bin {p5['bin']['ms']:.2f} ms, query {p5['query']['ms']:.2f} ms, unbin {p5['unbin']['ms']:.2f} ms. "
              f"Clock throttle reasons seen: config 3 {d3['clocks']['reasons'] or 'none'}, config 5 "
              f"{d5['clocks']['reasons'] or 'none'} (sw_power_cap is kept, as the rules allow).\n")
    p = os.path.join(ROOT, "DESIGN.md")
    s = open(p).read()
    a = s.index("| **3 (headline)** |")
    b = s.index("The reference arm (`bench.py --impl reference`, config 3)")
    s = s[:a] + table + "\n\n" + passes + "\n" + s[b:]
    a = s.index("* **Speed-ups over the reference's own multithreaded CPU query**")
    b = s.index("* **Launch list** of `bench.py")
    v, e, c, rv = d3["value"], d3["e2e"]["value"], d3["cpu_baseline"]["value"], r["value"]
    s = s[:a] + (f"* **Speed-ups over the reference's own multithreaded CPU query** at config 3: {v / c:.0f}×\n"
                 f"  device-resident, {e / c:.1f}× end to end against the in-line CPU baseline "
                 f"({v / rv:.0f}× / {e / rv:.1f}× against\n  the reference arm's run).\n") + s[b:]
    open(p, "w").write(s)

    p = os.path.join(ROOT, "README.md")
    lines = open(p).read().split("\n")
    rows = {
        "| config 3:": f"| config 3: 1e9 u64 keys, shuffled (partitioned path) | {v:.1f} Gkeys/s ({d3['ms_per_step']:.1f} ms), "
                       f"{d3['gather_roofline']['frac']:.2f}× the measured gather roofline, {d3['roofline']['frac']:.2f} of HBM | "
                       f"{e:.2f} Gkeys/s (PCIe-bound) | {c:.2f} Gkeys/s |",
        "| config 5:": f"| config 5: 1e9 k-mers, fused front end (partitioned path) | {d5['value']:.1f} Gkeys/s | "
                       f"{d5['e2e']['value']:.1f} Gkeys/s | {d5['cpu_baseline']['value']:.2f} Gkeys/s |",
        "| config 4:": f"| config 4: 3e8 strings | {d[4]['value']:.1f} Gkeys/s | {d[4]['e2e']['value']:.2f} Gkeys/s | "
                       f"{d[4]['cpu_baseline']['value']:.2f} Gkeys/s |",
        "| config 2:": f"| config 2: 1e8 queries, L2-resident pilots | {d[2]['value']:.0f} Gkeys/s | {d[2]['e2e']['value']:.2f} Gkeys/s | "
                       f"{d[2]['cpu_baseline']['value']:.2f} Gkeys/s |",
    }
    out = []
    for L in lines:
        for k, nv in rows.items():
            if L.startswith(k):
                L = nv
        out.append(L)
    open(p, "w").write("\n".join(out))


if __name__ == "__main__":
    main()
