"""Per-kernel totals from an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/launch_summary.py launches.csv [steps]"""
import collections
import csv
import sys


def main(path, steps=1):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if r[vi] in ("", "Metric Value"):
            continue
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r[ui], 1.0)
        name = r[ki].split("(")[0][:70]
        if "_probe" in name or "at::" in name:  # bench's roofline probes and torch's L2 flush: not the step
            continue
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    all_ms = sum(tot.values())
    print(f"total {all_ms / steps:.3f} ms per step over {sum(cnt.values())} launches ({steps} steps)")
    for k, v in tot.most_common(15):
        print(f"{v / steps:9.3f} ms  {cnt[k] / steps:6.1f}x  {100 * v / all_ms:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
