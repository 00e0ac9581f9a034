#!/usr/bin/env python
"""Write tests/golden/<cfg>_fit.json: the ORACLE's Newton fit (oracle/ only) of a BASELINE config.
Used by tests/test_gpu_parity.py::test_fit_parity_golden (identical iterations / halvings, coefs 1e-8)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle as O  # noqa: E402


def main(cfgs, tol=1e-6):
    for cfg in cfgs:
        t0 = time.time()
        prob = datagen.make(cfg)
        D = O.Data(prob.X, prob.Y, prob.Z, prob.choice, prob.spec.K)
        fit = O.newton_fit(D, tol=tol)
        out = dict(config=cfg, seed=0, tol=tol, status=fit.status, iters=fit.iters,
                   halvings=[h["halvings"] for h in fit.history], loglik=fit.loglik, grad_norm=fit.grad_norm,
                   history=fit.history, coef=[float(x) for x in fit.coef],
                   source="oracle/mnl_oracle.py newton_fit (tools/make_golden_fits.py)", seconds=time.time() - t0)
        path = os.path.join(ROOT, "tests", "golden", f"{cfg}_fit.json")
        with open(path, "w") as fh:
            json.dump(out, fh, indent=0)
        print(cfg, fit.status, fit.iters, out["halvings"], fit.loglik, f"{time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3", "c5"])
