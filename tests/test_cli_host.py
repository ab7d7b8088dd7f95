"""Host side of the regression-bench front end (paper_2511_16340_b200/cli.py): the dataset.cpp
restatement (load_csv errors, standardize, sample_split with the reference Rng), argument
defaults and the CSV header -- no GPU calls."""
import numpy as np
import pytest

from oracle import oracle as O


@pytest.fixture(scope="module")
def cli():
    from paper_2511_16340_b200 import cli as c
    return c


def test_csv_header_matches_reference(cli):
    # bench/regression.hpp:63-65
    assert cli.CSV_HEADER == ("trial,solver,system,init,iters,converged,final_rel_residual,"
                              "d_euclid_ratio,d_rkhs_ratio,identity_gap,seed")


def test_load_csv_and_errors(cli, tmp_path):
    p = tmp_path / "d.csv"
    p.write_text("x,y,t\n1, 2 ,3\n4,5,6\r\n\n7,8,9\n")
    X, y, name = cli.load_csv(str(p), 2, has_header=True)
    assert name == "d" and X.tolist() == [[1, 2], [4, 5], [7, 8]] and y.tolist() == [3, 6, 9]
    X, y, _ = cli.load_csv(str(p), 0, has_header=True)
    assert y.tolist() == [1, 4, 7] and X.tolist() == [[2, 3], [5, 6], [8, 9]]
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2\n3,x\n")
    with pytest.raises(cli.ParseError, match="bad.csv:2: non-numeric cell 'x'"):
        cli.load_csv(str(bad), 1)
    rag = tmp_path / "rag.csv"
    rag.write_text("1,2\n3,4,5\n")
    with pytest.raises(cli.ParseError, match="rag.csv:2: expected 2 cells, got 3"):
        cli.load_csv(str(rag), 1)
    with pytest.raises(cli.ParseError, match="target column 5 out of range"):
        cli.load_csv(str(rag), 5)
    with pytest.raises(cli.ParseError, match="cannot open"):
        cli.load_csv(str(tmp_path / "none.csv"), 0)


def test_standardize(cli):
    X = np.array([[1.0, 5.0], [3.0, 5.0], [5.0, 5.0]])
    y = np.array([2.0, 4.0, 9.0])
    Xs, ys = cli.standardize(X, y)
    np.testing.assert_allclose(Xs[:, 0], [-1.224744871391589, 0.0, 1.224744871391589])
    assert np.all(Xs[:, 1] == 0.0)  # constant column -> zeros
    assert abs(ys.mean()) < 1e-15 and abs(ys.std() - 1.0) < 1e-15


def test_sample_split_follows_reference_rng(cli):
    n, n1, n2, seed = 50, 20, 7, 1234
    X = np.arange(n, dtype=float)[:, None] * np.ones((1, 3))
    y = np.arange(n, dtype=float)
    X1, y1, X2, y2 = cli.sample_split(X, y, n1, n2, seed)
    # the partial Fisher-Yates of dataset.cpp:160-167 driven by the reference-pinned oracle Rng
    idx = list(range(n))
    r = O.Rng(seed)
    for i in range(n1 + n2):
        j = i + r.uniform_index(n - i)
        idx[i], idx[j] = idx[j], idx[i]
    assert y1.tolist() == idx[:n1] and y2.tolist() == idx[n1:n1 + n2]
    assert len(set(y1) | set(y2)) == n1 + n2
    with pytest.raises(ValueError):
        cli.sample_split(X, y, 40, 20, seed)


def test_thompson_host_helpers(cli):
    # radical inverse / Halton (thompson.cpp:93-124)
    assert cli.radical_inverse(1, 2) == 0.5 and cli.radical_inverse(6, 2) == 0.375
    assert cli.radical_inverse(5, 3) == pytest.approx(2 / 3 + 1 / 9, abs=0)
    assert [cli.nth_prime(k) for k in (0, 1, 5, 35, 36)] == [2, 3, 13, 151, 157]
    X = cli.init_design(3, 40, 7)
    assert X.shape == (40, 3) and np.all((X >= 0) & (X < 1))
    np.testing.assert_array_equal(X, cli.init_design(3, 40, 7))
    # the shift is the first draws of Rng(derive_seed(seed, 0xde5160))
    r = O.Rng(O.derive_seed(7, 0xDE5160))
    shift = [r.uniform() for _ in range(3)]
    v = cli.radical_inverse(1, 2) + shift[0]
    assert X[0, 0] == v - np.floor(v)
    # candidates: uniform share first, then softmax-anchored perturbations clamped to [0, 1]
    y = np.linspace(0.0, 1.0, 40)
    C = cli.propose_candidates(X, y, 20, 0.3, 0.25, 1.0, 11)
    assert C.shape == (20, 3) and np.all((C >= 0) & (C <= 1))
    r = O.Rng(11)
    assert C[0, 0] == r.uniform() and C[0, 1] == r.uniform()
    flat = cli.propose_candidates(X, np.zeros(40), 10, 0.3, 0.0, 1.0, 3)  # T = 0: all on the argmax
    r = O.Rng(3)
    r.uniform()
    assert flat[0, 0] == min(max(X[0, 0] + 0.15 * r.normal(), 0.0), 1.0)


def test_cli_arguments(cli):
    with pytest.raises(SystemExit):
        cli.main(["thompson-bench", "--budget", "medium"])
    assert cli.main(["regression-bench", "--data", "/nonexistent.csv", "--solvers", "cg"]) == 1
    assert cli.short_num(0.3) == "0.3" and cli.short_num(1e-5) == "1e-05" and cli.fmt(0.1) == "0.10000000000000001"
