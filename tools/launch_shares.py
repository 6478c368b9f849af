"""Per-kernel shares of an ncu launch list (`--metrics gpu__time_duration.sum --csv`), as a markdown table.

    python tools/launch_shares.py gpurun_out/<tag>_launches_cfg2.csv
"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        v *= {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        tot[name] += v
        cnt[name] += 1
    ours = {k: v for k, v in tot.items() if "chem::" in k}
    s = sum(ours.values())
    print("| kernel | launches | total ns | share of our kernels |")
    print("|---|---|---|---|")
    for k, v in sorted(ours.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.0f} | {100 * v / s:.2f}% |")
    other = sum(v for k, v in tot.items() if k not in ours)
    print(f"\nOther (torch copies for the restore, energy setup): {other:.0f} ns.")


if __name__ == "__main__":
    main(sys.argv[1])
