"""The reference-side plugin seam: ``paper_2102_05221_b200.speedups`` is a drop-in for
``elastik._speedups`` (pkg/src/elastik/_speedups.pyx:274-317), the module the reference's
``engines._dispatch`` (pkg/src/elastik/engines.py:29-50) calls once per pair.

tests/golden/dispatch.npz holds every ``_speedups.run`` call the LIVE reference issued while
its own public API ran (tests/golden/make_golden_dispatch.py): compute_base's ``window=0``,
windowed base, ea / eapruned with running and diagonal-bound cutoffs, infeasible windows and
``orient="st"`` recurrences with the shorter series on the rows.  The GPU replays them through
``speedups.run`` / ``run_many`` and must return the reference's (cost, cells) exactly.
"""

import math

import numpy as np
import pytest

from conftest import load_golden

ENGINES = ("base", "ea", "eapruned")


def calls():
    g = load_golden("dispatch.npz")
    cut = lambda name: np.split(g[name], np.cumsum(g[name + "_len"])[:-1])  # noqa: E731
    lines, cols, wts, vbs, hbs = cut("lines"), cut("cols"), cut("weights"), cut("vb"), cut("hb")
    out = []
    for k in range(len(g["engine"])):
        p = g["params"][k]
        out.append(dict(engine=str(g["engine"][k]), lines=np.ascontiguousarray(lines[k]),
                        cols=np.ascontiguousarray(cols[k]), kind=int(g["kind"][k]), mode=int(g["mode"][k]),
                        window=int(g["window"][k]), cutoff=float(g["cutoff"][k]), gap=float(p[0]), c=float(p[1]),
                        nu=float(p[2]), lam=float(p[3]), weights=np.ascontiguousarray(wts[k]),
                        vb=np.ascontiguousarray(vbs[k]), hb=np.ascontiguousarray(hbs[k]),
                        cost=float(g["cost"][k]), cells=int(g["cells"][k])))
    return out


def args_of(c):
    return (c["engine"], c["lines"], c["cols"], c["kind"], c["mode"], c["window"], c["cutoff"], c["gap"], c["c"],
            c["nu"], c["lam"], c["weights"], c["vb"], c["hb"])


def same(a, b):
    return (math.isnan(a) and math.isnan(b)) or a == b


def test_fixture_covers_the_seam_cases():
    cs = calls()
    assert {c["engine"] for c in cs} == set(ENGINES)
    base = [c for c in cs if c["engine"] == "base"]
    assert base and all(c["window"] == 0 for c in base if len(c["lines"]) >= len(c["cols"])), \
        "compute_base passes window=0 (engines.py:60-62)"
    assert any(len(c["lines"]) < len(c["cols"]) for c in cs), "orient='st' rows shorter than columns"
    assert any(c["cost"] == math.inf and c["cells"] == 0 for c in cs), "infeasible windows"
    assert len({c["kind"] for c in cs}) == 6


def test_oracle_run_matches_the_recorded_reference_calls():
    """The C restatement's run (oracle/ek_oracle.c) pins the fixture: same (cost, cells)."""
    from oracle import eko

    bad = []
    for c in calls():
        cost, cells = eko.run(*args_of(c))
        if not (same(cost, c["cost"]) and cells == c["cells"]):
            bad.append((c["engine"], len(c["lines"]), len(c["cols"]), c["kind"], cost, c["cost"], cells, c["cells"]))
    assert not bad, bad[:5]


def test_run_argument_errors_before_the_device():
    """run's argument checking mirrors the .pyx (no GPU needed: it raises before the ABI)."""
    from paper_2102_05221_b200 import speedups

    a = np.arange(5.0)
    with pytest.raises(KeyError):
        speedups.run("pruned_only", a, a, 0, 0, 5, math.inf, 0.0, 0.0, 0.0, 0.0, speedups.EMPTY, speedups.EMPTY,
                     speedups.EMPTY)
    with pytest.raises(ValueError):
        speedups.run("base", np.arange(5, dtype=np.float32), a, 0, 0, 5, math.inf, 0.0, 0.0, 0.0, 0.0,
                     speedups.EMPTY, speedups.EMPTY, speedups.EMPTY)
    with pytest.raises(ValueError):
        speedups.run("base", np.arange(10.0)[::2], a, 0, 0, 5, math.inf, 0.0, 0.0, 0.0, 0.0, speedups.EMPTY,
                     speedups.EMPTY, speedups.EMPTY)
    with pytest.raises(ValueError):  # wdtw without its weight table
        speedups.run("base", a, a, 2, 0, 5, math.inf, 0.0, 0.0, 0.0, 0.0, speedups.EMPTY, speedups.EMPTY,
                     speedups.EMPTY)
    with pytest.raises(NotImplementedError):  # custom borders on a kind without them
        speedups.run("base", a, a, 0, 0, 5, math.inf, 0.0, 0.0, 0.0, 0.0, speedups.EMPTY, np.zeros(6), np.zeros(6))
    with pytest.raises(NotImplementedError):  # erp borders that are not _erp_border's
        speedups.run("base", a, a, 3, 0, 5, math.inf, 0.0, 0.0, 0.0, 0.0, speedups.EMPTY, np.zeros(6), np.zeros(6))


@pytest.mark.gpu
def test_gpu_run_replays_every_recorded_call(gpu):
    """Batched: one run_many call per (engine, kind, mode, parameters) group."""
    from paper_2102_05221_b200 import speedups

    groups = {}
    for k, c in enumerate(calls()):
        key = (c["engine"], c["kind"], c["mode"], c["gap"], c["c"], c["nu"], c["lam"])
        groups.setdefault(key, []).append(k)
    cs = calls()
    bad, n = [], 0
    for (engine, kind, mode, gap, cc, nu, lam), ks in groups.items():
        # WDTW tables differ per g: split the group by table
        by_tab = {}
        for k in ks:
            by_tab.setdefault(cs[k]["weights"].tobytes() if kind == 2 else b"", []).append(k)
        for sub in by_tab.values():
            costs, cells = speedups.run_many(
                engine, [(cs[k]["lines"], cs[k]["cols"]) for k in sub], kind, mode,
                [cs[k]["window"] for k in sub], [cs[k]["cutoff"] for k in sub], gap, cc, nu, lam,
                weights=[cs[k]["weights"] for k in sub], borders=[(cs[k]["vb"], cs[k]["hb"]) for k in sub])
            for k, co, ce in zip(sub, costs.tolist(), cells.tolist()):
                n += 1
                if not (same(co, cs[k]["cost"]) and ce == cs[k]["cells"]):
                    bad.append((engine, kind, mode, len(cs[k]["lines"]), len(cs[k]["cols"]), cs[k]["window"],
                                cs[k]["cutoff"], co, cs[k]["cost"], ce, cs[k]["cells"]))
    assert n == len(cs)
    assert not bad, f"{len(bad)} of {n} mismatches: {bad[:5]}"


@pytest.mark.gpu
def test_gpu_run_single_calls(gpu):
    """The unbatched run() -- what _dispatch calls -- on a spread of the recorded calls."""
    from paper_2102_05221_b200 import speedups

    cs = calls()
    for c in cs[:: max(1, len(cs) // 150)]:
        cost, cells = speedups.run(*args_of(c))
        assert same(cost, c["cost"]) and cells == c["cells"], (c["engine"], c["kind"], cost, c["cost"], cells,
                                                               c["cells"])


@pytest.mark.gpu
def test_gpu_compute_functions_keep_st_orientation(gpu):
    """compute_ea / compute_eapruned on orient='st' recurrences equal the oracle's run on the
    same (unswapped) lines / cols, including ea's orientation-dependent row abandoning."""
    import paper_2102_05221_b200 as ekb
    from oracle import eko

    rng = np.random.default_rng(5)
    for kind in ekb.KINDS:
        for _ in range(6):
            la, lb = sorted(int(x) for x in rng.integers(2, 60, size=2))
            spec = {"dtw": ekb.DistanceSpec(kind="dtw"), "cdtw": ekb.DistanceSpec(kind="cdtw", window=5),
                    "wdtw": ekb.DistanceSpec(kind="wdtw", wdtw_g=0.1),
                    "erp": ekb.DistanceSpec(kind="erp", window=6, erp_gap=0.2),
                    "msm": ekb.DistanceSpec(kind="msm", msm_c=0.5),
                    "twe": ekb.DistanceSpec(kind="twe", twe_nu=0.01, twe_lambda=0.5)}[kind]
            s, t = np.cumsum(rng.normal(size=la)), np.cumsum(rng.normal(size=lb))
            rec = ekb.make_recurrence(spec, s, t, orient="st")
            assert rec.shape == (la, lb)
            w = int(rng.integers(0, lb + 2))
            wt = rec.wdtw_weights if rec.wdtw_weights is not None else np.empty(0)
            vb = rec.v_border_vals if rec.v_border_vals is not None else np.empty(0)
            hb = rec.h_border_vals if rec.h_border_vals is not None else np.empty(0)
            for co in (math.inf, 2.0, 25.0):
                for eng, fn in (("ea", ekb.compute_ea), ("eapruned", ekb.compute_eapruned)):
                    got = fn(rec, w, co)
                    want = eko.run(eng, rec.lines, rec.cols, ekb.KINDS.index(kind),
                                   0 if spec.cost_mode == "squared" else 1, w, co, spec.erp_gap or 0.0,
                                   spec.msm_c or 0.0, spec.twe_nu or 0.0, spec.twe_lambda or 0.0, wt, vb, hb)
                    assert (got.cost, got.cells_computed) == want, (kind, eng, la, lb, w, co, got, want)
            got = ekb.compute_base(rec)
            assert got.cells_computed == la * lb
