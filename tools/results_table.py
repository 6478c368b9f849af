"""Markdown results table from bench lines: python tools/results_table.py profiles/r01g"""
import json
import sys


def main(prefix):
    print("| config | Mcell-steps/s (1 B200) | e2e (host buffers) | ms/step | substeps per cell-step | "
          "FP64 roofline frac (algorithmic) | oracle, host cores | GPU/oracle |")
    print("|---|---|---|---|---|---|---|---|")
    for c in ("cfg2", "cfg3", "cfg4", "cfg5"):
        try:
            d = json.loads(open(f"{prefix}_bench_{c}.json").read().strip().splitlines()[-1])
        except OSError:
            continue
        cb = d.get("cpu_baseline") or {}
        ext = " (extrapolated)" if "extrapol" in (cb.get("sample", "") + cb.get("kind", "")).lower() else ""
        ratio = f"{d['value'] / cb['value']:.0f}x" if cb.get("value") else "-"
        print(f"| {c} | {d['value']:.1f} | {(d.get('e2e') or {}).get('value', float('nan')):.1f} | "
              f"{d['ms_per_step']:.1f} | {d['detail']['substeps_per_cell_step']:.2f} | "
              f"{d['roofline']['frac']:.3f} | {cb.get('value', float('nan')):.3f}{ext}, {cb.get('cores', '?')} cores | "
              f"{ratio} |")


if __name__ == "__main__":
    main(sys.argv[1])
