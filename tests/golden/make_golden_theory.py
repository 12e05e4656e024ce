"""Golden vectors for the host-side threshold study, produced by the REAL
reference (`cutbench.costmodel`, `cutbench.svmfit`, `cutbench.harness.
detect_crossovers`, `cutbench.cli` threshold). Run in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_theory.py

Writes tests/golden/reference_theory.json. The fit datasets are seeded
synthetic (q, c_total, delta) grids shaped like a threshold sweep: a noisy
linear boundary plus clipped outliers, so the weight clipping and both label
classes are exercised.
"""
from __future__ import annotations

import io
import json
import os
from contextlib import redirect_stdout

import numpy as np

from cutbench import cli, costmodel, harness, svmfit  # the reference, via PYTHONPATH
from cutbench.errors import DegenerateFitError, ValidationError

HERE = os.path.dirname(os.path.abspath(__file__))


def fit_dataset(seed, slope, icpt, qs, cs, noise):
    rng = np.random.default_rng(seed)
    pts, dl = [], []
    for q in qs:
        for c in cs:
            d = (c - (slope * q + icpt)) * 0.3 + rng.normal(0, noise)
            if rng.uniform() < 0.05:
                d *= 40.0
            pts.append([q, c])
            dl.append(d)
    return np.array(pts, float), np.array(dl)


def main():
    out = {"threshold_line": {}, "threshold_uniform": [], "n_sub": [], "regime": [], "predict": [],
           "nonuniform": [], "fits": [], "errors": {}, "cli_threshold": [], "crossovers": []}
    for n in range(2, 9):
        out["threshold_line"][str(n)] = list(costmodel.threshold_line(n))
    for q, n, c in [(24, 2, 6), (24, 2, 12), (24, 3, 4), (30, 3, 20), (32, 4, 4), (20, 4, 17), (12, 2, None)]:
        r = costmodel.threshold_uniform(q, n, c)
        out["threshold_uniform"].append({"args": [q, n, c], "c_total_max": r.c_total_max, "slope": r.slope,
                                         "delta": r.delta, "satisfied": r.satisfied})
    for n, c, k in [(2, 3, 2), (3, 2, 2), (4, 1, 2), (5, 3, 3)]:
        out["n_sub"].append({"args": [n, c, k], "value": costmodel.n_sub_uniform(n, c, k)})
    for q, n, c, d, ds in [(24, 2, 6, 30.0, 15.0), (12, 3, 1, 8.0, 4.0), (30, 2, 2, 20.0, 20.0),
                           (8, 4, 3, 40.0, 10.0), (16, 2, 14, 10.0, 5.0)]:
        p = costmodel.CostParams(q=q, n=n, c=c, depth=d, seg_depth=ds)
        rr = costmodel.regime_ratios(p)
        out["regime"].append({"args": [q, n, c, d, ds], "r_pre_sub": rr.r_pre_sub, "r_pre_merge": rr.r_pre_merge,
                              "r_sub_merge": rr.r_sub_merge, "regime": rr.regime})
        ns = costmodel.n_sub_uniform(n, c)
        out["predict"].append({"args": [q, n, c, d, ds, ns], "value": list(costmodel.predict_costs(p, ns))})
        out["nonuniform"].append({"args": [q, n, c, d, ds, ns], "value": costmodel.threshold_nonuniform(p, ns)})
    for bad in [dict(q=4, n=1, c=1, depth=1.0, seg_depth=1.0), dict(q=4, n=2, c=1, depth=4.0, seg_depth=1.0),
                dict(q=4, n=2, c=1, depth=4.0, seg_depth=2.0, k=1)]:
        try:
            costmodel.CostParams(**bad)
            out["errors"][json.dumps(bad)] = "ok"
        except ValidationError as e:
            out["errors"][json.dumps(bad)] = type(e).__name__
    for seed, (slope, icpt, qs, cs, noise, init, iters) in enumerate([
        (0.5, 0.0, range(2, 21, 2), range(1, 11), 0.2, (0.5, 0.0), 10_000),
        (0.7, -7.3, range(12, 31, 2), range(1, 15), 0.5, (0.5, 0.0), 10_000),
        (0.66, 1.6, range(3, 19, 3), range(2, 13, 2), 0.1, (2 / 3, 1.58), 10_000),
        (0.4, 2.0, range(10, 30, 4), range(1, 12), 0.3, (0.5, 0.0), 500),
    ]):
        pts, dl = fit_dataset(seed, slope, icpt, qs, cs, noise)
        f = svmfit.fit_weighted_line(pts, dl, init, iterations=iters)
        out["fits"].append({"points": pts.tolist(), "deltas": dl.tolist(), "init": list(init), "iterations": iters,
                            "slope": f.slope, "intercept": f.intercept, "w": f.w.tolist(), "b": f.b,
                            "weighted_accuracy": f.weighted_accuracy, "margin_violations": f.margin_violations,
                            "weights": f.weights.tolist()})
    try:
        svmfit.fit_weighted_line(np.array([[2.0, 1.0], [4.0, 1.0]]), np.array([-1.0, -2.0]), (0.5, 0.0))
    except DegenerateFitError as e:
        out["errors"]["one_class"] = type(e).__name__
    for argv in (["threshold", "--q", "24", "--n", "3", "--c", "4"], ["threshold", "--q", "20", "--c", "7"],
                 ["threshold", "--q", "24", "--n", "4", "--c", "5"]):
        buf = io.StringIO()
        with redirect_stdout(buf):
            rc = cli.main(argv)
        out["cli_threshold"].append({"argv": argv, "rc": rc, "json": json.loads(buf.getvalue())})
    TB = harness.TimingBreakdown
    series = [TB(q, 2, 6, 10, 100, pre, sub, mer, pre + sub + mer, 1.0, 0.0, 1, st)
              for q, pre, sub, mer, st in [(10, 1e-3, 2e-3, 1e-4, "ok"), (12, 1e-3, 2e-3, 2e-3, "ok"),
                                            (14, 1e-3, 2e-3, 2.5e-3, "timeout-cut"), (16, 1e-3, 2e-3, 9e-3, "ok")]]
    c = harness.detect_crossovers(series)
    out["crossovers"].append({"rows": [[b.q, b.t_pre, b.t_sub, b.t_merge, b.status] for b in series],
                              "q_pre_cross": c.q_pre_cross, "q_sub_cross": c.q_sub_cross})
    with open(os.path.join(HERE, "reference_theory.json"), "w") as fh:
        json.dump(out, fh, indent=0, allow_nan=False)
    print("wrote", os.path.join(HERE, "reference_theory.json"))


if __name__ == "__main__":
    main()
