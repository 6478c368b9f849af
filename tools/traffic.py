"""profiles/traffic.json from ncu CSVs of the k_integrate launches of one bench run per config
(dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged over the run's launches, weighted
like the bench's `achieved`: total bytes / launches) plus the launch-list share of k_integrate.

    python tools/traffic.py TAG cfg2 cfg3 ...     (reads gpurun_out/TAG_traffic_<cfg>.csv)
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(tag, *cfgs):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    doc = json.load(open(path)) if os.path.exists(path) else {}
    for c in cfgs:
        rows = [r for r in csv.reader(open(os.path.join(ROOT, "gpurun_out", f"{tag}_traffic_{c}.csv")))
                if len(r) > 10 and r[0].isdigit()]
        per = {}
        for r in rows:
            per.setdefault(r[0], {})[r[12]] = float(r[14].replace(",", ""))
        ks = [v for v in per.values()]
        unit = {}
        for r in rows:
            unit[r[12]] = r[13]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = sum(v["dram__bytes_read.sum"] * scale[unit["dram__bytes_read.sum"]] +
                  v["dram__bytes_write.sum"] * scale[unit["dram__bytes_write.sum"]] for v in ks)
        keep = {k: v for k, v in doc.get(c, {}).items() if k.startswith("ncu_")}   # FP64-pipe % from full captures
        doc[c] = {"traffic_bytes_per_launch": tot / max(len(ks), 1), "launches": len(ks),
                  "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every k_integrate "
                            f"launch of `bench.py --config {c} --steps 1 --warmup 3` (gpurun {tag})", **keep}
        print(c, doc[c])
    json.dump(doc, open(path, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
