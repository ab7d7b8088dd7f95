"""The regression-bench front end (paper_2511_16340_b200/cli.py) on the device:
the reference's CSV header and row layout, the config sidecar, the protocol's invariants
(cold rows carry distance ratios 1, warm rows the report's; the identity gap of the Schur
route is at rounding level), and the warm start's effect on the posterior-mean system."""
import csv
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_regression_bench_cli(tmp_path):
    from paper_2511_16340_b200 import cli

    rng = np.random.default_rng(5)
    n, d = 400, 4
    X = rng.random((n, d))
    yv = np.sin(3 * X[:, 0]) + X[:, 1] ** 2 + 0.05 * rng.standard_normal(n)
    path = tmp_path / "toy.csv"
    np.savetxt(path, np.column_stack([X, yv]), delimiter=",", header="a,b,c,d,y", comments="")
    out = tmp_path / "out"
    rc = cli.main(["regression-bench", "--data", str(path), "--has-header", "--n1", "200", "--n2", "40",
                   "--trials", "2", "--tol", "1e-4", "--mll-steps", "10", "--features", "256",
                   "--sgd-lr-grid", "0.01,0.03", "--sgd-max-iters", "3000", "--out", str(out)])
    assert rc == 0
    rows = list(csv.reader(open(out / "regression_toy.csv")))
    assert ",".join(rows[0]) == cli.CSV_HEADER
    body = rows[1:]
    assert len(body) == 2 * 2 * 3 * 2  # trials x systems x solvers x inits
    for r in body:
        rec = dict(zip(rows[0], r))
        assert rec["solver"] in ("cg", "sgd", "ap") and rec["system"] in ("mean", "sample")
        if rec["init"] == "cold":
            assert float(rec["d_euclid_ratio"]) == 1.0 and float(rec["d_rkhs_ratio"]) == 1.0
        else:
            assert 0.0 <= float(rec["d_rkhs_ratio"]) < 1.0
        assert abs(float(rec["identity_gap"])) < 1e-6
    cg = [dict(zip(rows[0], r)) for r in body if r[1] == "cg"]
    assert all(r["converged"] == "1" for r in cg)
    warm = np.mean([int(r["iters"]) for r in cg if r["init"] == "warm"])
    cold = np.mean([int(r["iters"]) for r in cg if r["init"] == "cold"])
    assert warm <= cold
    side = open(out / "regression_toy.config.txt").read()
    assert side.startswith("command=regression-bench\ndataset=toy\n") and "config_hash=" in side


def test_thompson_bench_cli(tmp_path):
    """thompson-bench: one CSV per (lengthscale, seed, init) with the reference's header and a
    row per (solver, round); round 0 is the initial design (NaN residuals); the best value
    never decreases; warm and cold share the objective and the initial design (same round-0
    best); two runs with the same seeds agree except for wall-clock time."""
    from paper_2511_16340_b200 import cli

    def run(out):
        rc = cli.main(["thompson-bench", "--dim", "2", "--n-init", "60", "--samples", "4", "--rounds", "3",
                       "--lengthscales", "0.3", "--seeds", "1", "--solvers", "cg,ap", "--proposal-count", "64",
                       "--proposal-rounds", "2", "--ascent-steps", "5", "--features", "256", "--out", str(out)])
        assert rc == 0

    run(tmp_path / "a")
    run(tmp_path / "b")
    files = sorted(os.listdir(tmp_path / "a"))
    assert files == ["thompson.config.txt", "thompson_l0.3_s0_cold.csv", "thompson_l0.3_s0_warm.csv"]
    firsts = {}
    for fn in files[1:]:
        ra = list(csv.reader(open(tmp_path / "a" / fn)))
        rb = list(csv.reader(open(tmp_path / "b" / fn)))
        assert ",".join(ra[0]) == cli.THOMPSON_CSV_HEADER
        assert len(ra) == 1 + 2 * 4  # solvers x (rounds + 1)
        for x, y in zip(ra[1:], rb[1:]):
            assert x[:8] == y[:8]  # everything but wall_clock_s
        for solver in ("cg", "ap"):
            rows = [r for r in ra[1:] if r[2] == solver]
            assert [int(r[0]) for r in rows] == [0, 1, 2, 3]
            assert rows[0][6] == "nan" and rows[0][7] == "nan"
            best = [float(r[5]) for r in rows]
            assert all(b2 >= b1 for b1, b2 in zip(best, best[1:]))
            firsts.setdefault(solver, set()).add(rows[0][5])
    assert all(len(v) == 1 for v in firsts.values())  # matched warm/cold pairs
