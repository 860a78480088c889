"""Golden fixtures for the host utilities of the drop-in API, from the LIVE reference:

    python tests/golden/make_golden_utils.py      (run in the build container)

utils.npz -- build_envelope / lb_keogh / lb_keogh2 on random series and windows,
derivative, gen_random_walk, and a load_tsv of a written file.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import refpkg  # noqa: E402

ek = refpkg.load()
assert ek is not None, "reference package not found"


def main():
    rng = np.random.default_rng(777)
    out = {}
    n_cases = 60
    lens = rng.integers(1, 70, size=n_cases)
    wins = [int(rng.integers(0, n + 3)) for n in lens]
    modes = ["squared" if rng.random() < 0.5 else "absolute" for _ in range(n_cases)]
    S = [np.cumsum(rng.normal(0, 1.5, n)) for n in lens]
    T = [np.cumsum(rng.normal(0, 1.5, n)) for n in lens]
    up, lo, lb, lb2, cuts = [], [], [], [], []
    for s, t, w, m in zip(S, T, wins, modes):
        es, et = ek.build_envelope(s, w), ek.build_envelope(t, w)
        up.append(es.upper)
        lo.append(es.lower)
        lb.append(ek.lb_keogh(t, es, m))
        cuts.append(float(rng.choice([np.inf, 1.0, 10.0])))
        lb2.append(ek.lb_keogh2(t, s, es, et, cutoff=cuts[-1], cost_mode=m))
    out["lens"] = lens
    out["wins"] = np.array(wins)
    out["modes"] = np.array([m == "squared" for m in modes])
    out["S"] = np.concatenate(S)
    out["T"] = np.concatenate(T)
    out["upper"] = np.concatenate(up)
    out["lower"] = np.concatenate(lo)
    out["lb"] = np.array(lb)
    out["lb2"] = np.array(lb2)
    out["lb2_cut"] = np.array(cuts)
    d = rng.normal(0, 1, 50)
    out["deriv_in"] = d
    out["deriv_out"] = ek.derivative(d)
    ds = ek.gen_random_walk(9, 31, 4, seed=12)
    out["rw_labels"] = np.array(ds.labels)
    out["rw_series"] = np.stack(ds.series)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "x.tsv")
        ek.write_tsv(ds, path, delimiter="comma")
        with open(path, encoding="utf-8") as fh:
            out["tsv_text"] = np.array(fh.read())
    np.savez_compressed(os.path.join(HERE, "utils.npz"), **out)


if __name__ == "__main__":
    main()
