"""c* (largest c_total with delta < 0) per (q, d) from sweep CSVs (the
reference CSV schema), plus the boundary fits next to them:
    python tools/boundary_table.py profiles/r01_boundary_native_d{5,10,20}.csv"""
import csv
import json
import os
import sys


def cstar(path):
    rows = list(csv.DictReader(open(path)))
    best = {}
    for r in rows:
        q, c, delta = int(r["q"]), int(r["c_total"]), float(r["delta"])
        best.setdefault(q, {})[c] = delta
    out = {}
    for q, by_c in sorted(best.items()):
        wins = [c for c, dl in sorted(by_c.items()) if dl < 0]
        # largest c such that every c' <= c wins (the contiguous speedup region)
        k = 0
        for c in sorted(by_c):
            if by_c[c] < 0:
                k = c
            else:
                break
        out[q] = (k, max(wins) if wins else 0)
    return out


def main():
    for path in sys.argv[1:]:
        tab = cstar(path)
        fit_path = path.replace(".csv", "_fit.json")
        fit = json.load(open(fit_path)) if os.path.exists(fit_path) else None
        line = " ".join(f"q={q}:{k}" for q, (k, _) in tab.items())
        extra = f"  fit c* = {fit['slope']:.3f} q {fit['intercept']:+.2f} (acc {fit['weighted_accuracy']:.3f})" if fit else ""
        print(f"{os.path.basename(path)}: {line}{extra}")


if __name__ == "__main__":
    main()
