"""Reference outputs of the equilibration diagnostics (check_equilibrated,
equilibration_objective; equilibration.py:227-287) on the matrices of
equil.npz at the reference's own d, e, and the on_sweep(k, d, e) sequence of
equilibrate on each (equil_sweeps.npz) (run where /root/reference exists):

    python tests/golden/make_golden_diag.py
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import graphform as gf  # noqa: E402  (the reference)

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    z = np.load(os.path.join(HERE, "equil.npz"))
    names = sorted({k.rsplit("_", 1)[0] for k in z.files if k.endswith("_A")})
    out = {}
    for name in names:
        A, d, e, gam = z[f"{name}_A"], z[f"{name}_d"], z[f"{name}_e"], float(z[f"{name}_gamma"])
        for tag, (dd, ee) in {"eq": (d, e), "even": (z[f"{name}_rd"], z[f"{name}_re"]),
                              "ones": (np.ones_like(d), np.ones_like(e))}.items():
            rep = gf.check_equilibrated(A, dd, ee, tol=0.05).as_dict()
            rep["objective"] = gf.equilibration_objective(A, dd, ee, gam)
            out[f"{name}|{tag}"] = rep
    sweeps = {}
    for name in names:
        rec = []
        gf.equilibrate(z[f"{name}_A"], on_sweep=lambda k, d, e: rec.append((k, d.copy(), e.copy())))
        sweeps[f"{name}_k"] = np.array([r[0] for r in rec])
        for k, d, e in rec:
            sweeps[f"{name}_d{k}"] = d
            sweeps[f"{name}_e{k}"] = e
    np.savez_compressed(os.path.join(HERE, "equil_sweeps.npz"), **sweeps)
    with open(os.path.join(HERE, "equil_diag.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(f"wrote equil_diag.json ({len(out)} reports)")


if __name__ == "__main__":
    main()
