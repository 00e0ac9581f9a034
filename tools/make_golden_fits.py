#!/usr/bin/env python
"""Write tests/golden/<cfg>_fit.json (numpy oracle) or <cfg>_fit_c.json (--c: the plain C oracle,
liboracle.so, with the full R7 margin log): the ORACLE's Newton fit (oracle/ only) of a BASELINE config.
Used by tests/test_gpu_parity.py::test_fit_parity_golden (identical iterations / halvings, coefs 1e-8)
and tests/test_golden_audit.py (the two oracles' fits agree; the R7 margin audit)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle as O  # noqa: E402
from oracle import coracle as OC  # noqa: E402


def main(cfgs, tol=1e-6, use_c=False):
    mod = OC if use_c else O
    for cfg in cfgs:
        t0 = time.time()
        prob = datagen.make(cfg)
        D = O.Data(prob.X, prob.Y, prob.Z, prob.choice, prob.spec.K)
        fit = mod.newton_fit(D, tol=tol)
        src = ("oracle/oracle.c oracle_mnl_newton_fit_log" if use_c else "oracle/mnl_oracle.py newton_fit")
        out = dict(config=cfg, seed=0, tol=tol, status=fit.status, iters=fit.iters,
                   halvings=[h["halvings"] for h in fit.history], loglik=fit.loglik, grad_norm=fit.grad_norm,
                   history=fit.history, coef=[float(x) for x in fit.coef],
                   source=src + " (tools/make_golden_fits.py)", seconds=time.time() - t0,
                   threads=OC.set_threads(0) if use_c else None)
        path = os.path.join(ROOT, "tests", "golden", f"{cfg}_fit{'_c' if use_c else ''}.json")
        with open(path, "w") as fh:
            json.dump(out, fh, indent=0)
        print(cfg, fit.status, fit.iters, out["halvings"], fit.loglik, f"{time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(args or ["c3", "c5"], use_c="--c" in sys.argv)
