"""Build profiles/ncu_summary.json (bench.py's roofline `traffic` source) from
`ncu --set full` raw CSV exports: profiles/<round>/ncu_full_<workload>.raw.csv.
usage: python tools/ncu_summarize.py profiles/r01c"""
import csv, json, os, re, sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0}


def val(s, unit=""):
    s = s.replace(",", "").strip()
    try:
        return float(s) * UNITS.get(unit.strip(), 1.0)
    except ValueError:
        return None


def summarize(path, rnd):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    # the heaviest launch in the capture
    best = max(rows[2:], key=lambda r: val(r[h.index("gpu__time_duration.sum")], units[h.index("gpu__time_duration.sum")]) or 0)
    g = lambda k: val(best[h.index(k)], units[h.index(k)]) if k in h else None
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    return {
        "kernel": re.sub(r"\(.*", "", best[h.index("Kernel Name")]),
        "dram_bytes_per_launch": (rd or 0) + (wr or 0),
        "dram_read_bytes": rd,
        "dram_write_bytes": wr,
        "duration_s": g("gpu__time_duration.sum"),
        "alu_pipe_pct": g("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "inst_executed": g("smsp__inst_executed.sum"),
        "registers": g("launch__registers_per_thread"),
        "grid": best[h.index("Grid Size")].strip("() ").split(",")[0],
        "block": best[h.index("Block Size")].strip("() ").split(",")[0],
        "source": f"{path} (ncu --set full --clock-control none, {rnd})",
    }


def main():
    d = sys.argv[1]
    out = {}
    for f in sorted(os.listdir(d)):
        m = re.match(r"ncu_full_(\w+)\.raw\.csv$", f)
        if m:
            out[m.group(1)] = summarize(os.path.join(d, f), os.path.basename(d.rstrip("/")))
    json.dump(out, open("profiles/ncu_summary.json", "w"), indent=1)
    for k, v in out.items():
        print(k, v["kernel"], f"{v['duration_s'] * 1e3:.3f} ms", f"{v['dram_bytes_per_launch'] / 1e6:.1f} MB")


if __name__ == "__main__":
    main()
