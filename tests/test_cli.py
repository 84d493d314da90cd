"""The B200 CLI (paper_1710_05781_b200/cli.py), mirroring the reference's
disctree CLI (cli.py:33-439): exit codes, input validation, 17-digit CSV.
CPU tests cover everything before the first device call; the GPU tests run
the commands end to end against the public API."""

import csv
import json

import numpy as np
import pytest

from paper_1710_05781_b200 import cli


def test_fmt17_round_trips():
    rng = np.random.default_rng(0)
    for v in np.concatenate([rng.normal(size=200) * 10.0 ** rng.integers(-300, 300, 200),
                             [0.1, 1 / 3, -2.5, 5e-324, 1.7976931348623157e308]]):
        assert float(cli.fmt17(v)) == v


def test_bad_arguments_exit_2(capsys):
    with pytest.raises(SystemExit) as e:
        cli.main(["evaluate", "--theta", "1.5"])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["bench", "--sizes", "10,x"])
    assert e.value.code == 2


@pytest.mark.parametrize("body,msg", [
    ("a,b\n1,2\n", "expected header"),
    ("x,q\n1,2,3\n", "line 2: expected 2 field"),
    ("x,q\n0.5,1\nfoo,2\n", "line 3: non-numeric"),
    ("x,q\n0.5,inf\n", "non-finite"),
])
def test_malformed_particles_exit_3(tmp_path, capsys, body, msg):
    f = tmp_path / "p.csv"
    f.write_text(body)
    assert cli.main(["evaluate", "--particles", str(f)]) == cli.EXIT_DATA
    assert msg in capsys.readouterr().err


def test_missing_inputs_exit_3(tmp_path, capsys):
    assert cli.main(["evaluate", "--particles", str(tmp_path / "nope.csv")]) == cli.EXIT_DATA
    assert cli.main(["evaluate"]) == cli.EXIT_DATA  # no source given
    assert "exactly one of" in capsys.readouterr().err
    d = tmp_path / "d.json"
    d.write_text(json.dumps({"domain": [0, 1], "cells": 2}))
    assert cli.main(["evaluate", "--density", str(d)]) == cli.EXIT_DATA
    assert "missing fields" in capsys.readouterr().err


def test_targets_reader(tmp_path):
    f = tmp_path / "t.csv"
    f.write_text("y\n0.25\n\n-1e-3\n")
    np.testing.assert_array_equal(cli.read_targets(str(f)), [0.25, -1e-3])


@pytest.mark.gpu
def test_evaluate_end_to_end(tmp_path, capsys):
    import paper_1710_05781_b200 as dt

    rng = np.random.default_rng(5)
    x, q = rng.uniform(-1, 1, 3000), rng.normal(size=3000)
    p = tmp_path / "p.csv"
    p.write_text("x,q\n" + "".join(f"{cli.fmt17(a)},{cli.fmt17(b)}\n" for a, b in zip(x, q)))
    t = tmp_path / "t.csv"
    ys = rng.uniform(-1.2, 1.2, 500)
    t.write_text("y\n" + "".join(f"{cli.fmt17(v)}\n" for v in ys))
    out = tmp_path / "e.csv"
    assert cli.main(["evaluate", "--particles", str(p), "--targets", str(t), "--rd", "0.01",
                     "--adaptive", "--tol", "1e-10", "--p", "8", "--out", str(out)]) == 0
    summary = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert summary["n_charges"] == 3000 and summary["method"] == "tree"
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["y", "E"]
    got = np.array([[float(a), float(b)] for a, b in rows[1:]])
    np.testing.assert_array_equal(got[:, 0], ys)
    system = dt.from_particles(np.column_stack([x, q]))
    k = dt.DiscKernel(0.01)
    cfg = dt.EvalConfig(p=8, adaptive=True, tolerance=1e-10)
    want = dt.evaluate_all(dt.build(system, k, cfg), k, cfg, system, ys).values
    np.testing.assert_array_equal(got[:, 1], want)  # 17 digits: bit-exact round trip


@pytest.mark.gpu
def test_accuracy_presets(tmp_path):
    out = tmp_path / "a.json"
    assert cli.main(["accuracy", "--table1", "--format", "json", "--out", str(out)]) == 0
    recs = json.load(open(out))
    assert [r["p"] for r in recs] == list(cli.TABLE1_PS)
    errs = [r["relative_error"] for r in recs]
    assert all(a > b for a, b in zip(errs, errs[1:]))  # decays with p (Table 1)
    assert cli.main(["accuracy", "--n", "5000", "--p", "20", "--out", str(tmp_path / "b.csv")]) == 0
    rows = list(csv.DictReader(open(tmp_path / "b.csv")))
    assert float(rows[0]["avg_relative"]) < 1e-11  # test_tree.py:280-289
