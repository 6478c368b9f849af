"""Print the key numbers of a bench JSON line (last line of the file)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable", e)
        continue
    rf = d.get("roofline") or {}
    print(path, "value=%.1f ms=%.2f frac=%.3f e2e=%s cpu=%s lpt=%s acc=%s sparse=%s clk=%s" % (
        d["value"], d["ms_per_step"], rf.get("frac", 0), (d.get("e2e") or {}).get("value"),
        (d.get("cpu_baseline") or {}).get("value"), d["detail"]["lpt"], d["detail"].get("hint_accuracy"),
        d["detail"]["sparse_cells"], (d.get("clocks") or {}).get("sm_mhz")))
    for k, v in (d.get("schedules") or {}).items():
        print("   ", k, "value=%.1f ms=%.1f frac=%.3f lpt=%s acc=%s" % (v["value"], v["ms_per_step"], v["frac"], v["lpt"],
                                                                  v.get("hint_accuracy")))
    if d.get("production_tolerance"):
        p = d["production_tolerance"]
        print("    production tol value=%.1f frac=%.3f substeps=%.2f" % (p["value"], p["frac"], p["substeps_per_cell_step"]))
    for a in d.get("also") or []:
        print("   also", a["config"], "value=%.1f ms=%.1f frac=%.3f lpt=%s acc=%s" % (
            a["value"], a["ms_per_step"], a["frac"], a["lpt"], a.get("hint_accuracy")))
        for k, v in (a.get("schedules") or {}).items():
            print("      ", k, "value=%.1f ms=%.1f frac=%.3f lpt=%s" % (v["value"], v["ms_per_step"], v["frac"], v["lpt"]))
