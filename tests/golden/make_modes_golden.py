"""Golden outcomes of the reference's condition-number mode and
target="closest" solves (run in the build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_modes_golden.py

Matrices come from oracle/gen.py (pinned to the reference generators in
generators.json), so the GPU box can rebuild them.  Writes
tests/golden/modes.json.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REF, "src"))

import itersvd  # noqa: E402
from itersvd.matio import SparseMatrixCsr  # noqa: E402

from oracle import gen as ogen  # noqa: E402


def cond_cases():
    """name -> (matrix spec, cfg kwargs) -- specs rebuilt by tests."""
    out = {}
    for kappa in (10.0, 1e2, 1e3):
        for seed in (2400, 2401):
            out["crit9_k%g_s%d" % (kappa, seed)] = ({"kind": "crit9", "kappa": kappa, "seed": seed},
                                                     {"seed": seed})
    out["diag5"] = ({"kind": "diag", "d": [1.0, 2.0, 3.0, 4.0, 5.0]}, {})
    out["zero_col_60x40"] = ({"kind": "zero_col", "m": 60, "n": 40, "col": 7, "seed": 14}, {})
    out["starved"] = ({"kind": "synth", "lo": 1e-2, "p": 30, "m": 50, "n": 30, "seed": 13},
                      {"max_matvecs": 30})
    out["sparse1003"] = ({"kind": "sparse", "seed": 1003}, {"seed": 0})
    return out


def closest_cases():
    return {
        "diag7": ({"kind": "diag", "d": [1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0]},
                  {"num_svals": 2, "target_values": [3.4, 6.2], "eps": 1e-9}),
        "synth2200": ({"kind": "synth", "lo": 1e-3, "p": 60, "m": 90, "n": 60, "seed": 2200},
                      {"num_svals": 2, "target_values": [0.05, 0.3], "eps": 1e-10, "seed": 2200}),
        "sparse1003": ({"kind": "sparse", "seed": 1003},
                       {"num_svals": 3, "target_values": [1.0, 2.0, 2.5], "eps": 1e-10, "seed": 3}),
    }


def _stats(s):
    return {"stage1_matvecs": s.stage1_matvecs, "stage2_matvecs": s.stage2_matvecs,
            "restarts": s.restarts, "resets": s.resets}


def main():
    out = {"cond": {}, "closest": {}}
    for name, (spec, kw) in cond_cases().items():
        m, n, rp, ci, va = ogen.build_spec(spec)
        a = SparseMatrixCsr(m, n, rp, ci, va)
        r = itersvd.estimate_condition_number(a, cfg=itersvd.SvdsConfig(**kw))
        out["cond"][name] = {"spec": spec, "cfg": kw, "kappa": float(r.kappa), "sigma_max": r.sigma_max,
                             "sigma_min": r.sigma_min, "infinite": bool(r.infinite),
                             "lower_bound": bool(r.lower_bound), "stats": _stats(r.stats)}
        print(name, r.kappa, r.infinite, r.lower_bound)
    for name, (spec, kw) in closest_cases().items():
        m, n, rp, ci, va = ogen.build_spec(spec)
        a = SparseMatrixCsr(m, n, rp, ci, va)
        res = itersvd.svds_solve(a, cfg=itersvd.SvdsConfig(target="closest", **kw))
        out["closest"][name] = {"spec": spec, "cfg": kw, "sigma": res.sigma.tolist(),
                                "rnorms": res.rnorms.tolist(), "converged": [bool(c) for c in res.converged],
                                "status": res.status, "stats": _stats(res.stats)}
        print(name, res.sigma, res.status)
    with open(os.path.join(HERE, "modes.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
