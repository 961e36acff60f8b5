"""The batched fitter (lowering.fit_linear_many / fit_for_grid_many) returns exactly what the
per-list fit_linear / fit_for_grid return (costmodel.py:93-141, 253-279): coefficients,
intercept and fit statistics bit for bit, the same FitError (message, collinear features),
the same quality warnings -- on every grid of the bench workloads' profile databases and on
random grids with collinear, constant, tiny and huge columns."""

from __future__ import annotations

import sys
import warnings
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _same(a, b):
    from paper_2002_06790_b200.errors import FitError

    if isinstance(a, FitError) or isinstance(b, FitError):
        return (type(a), str(a), getattr(a, "collinear_features", None)) == \
               (type(b), str(b), getattr(b, "collinear_features", None))
    return repr(a) == repr(b) and a.coefficients == b.coefficients and a.intercept == b.intercept \
        and a.fit_stats == b.fit_stats


def _per_list(recs):
    from paper_2002_06790_b200.errors import FitError
    from paper_2002_06790_b200.lowering import fit_linear

    try:
        return fit_linear(recs)
    except FitError as e:
        return e


def _all_groups(db):
    out = []
    for key in sorted(db.op_records):
        grid_map = db.op_records[key]
        groups = {}
        for k in sorted(grid_map):
            rec = grid_map[k]
            groups.setdefault(tuple(n for n, _ in rec.signature.arg_features), []).append(rec)
        out += list(groups.values())
    return out


def _dbs():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2002_06790_b200 import workloads as W

    yield "dag", W.dag_profiles(["hwA", "hwB"])
    yield "cnn", W.planted_profiles(W.CNN_LAWS)
    for wl in ("resnet50-dp8", "bert-large-ps-ar", "vgg16-sweep"):
        yield wl, bench.build_workload(0, 64, wl)[1]


@pytest.mark.parametrize("name", ["dag", "cnn", "resnet50-dp8", "bert-large-ps-ar", "vgg16-sweep"])
def test_workload_grids(name):
    from paper_2002_06790_b200.lowering import fit_for_grid, fit_for_grid_many, fit_linear_many

    db = dict(_dbs())[name]
    groups = _all_groups(db)
    assert groups
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        many = fit_linear_many(groups)
        for recs, m in zip(groups, many):
            assert _same(m, _per_list(recs))
    pairs = sorted(db.op_records)
    with warnings.catch_warnings(record=True) as w_one:
        warnings.simplefilter("always")
        one = {p: fit_for_grid(db, *p) for p in pairs}
    with warnings.catch_warnings(record=True) as w_many:
        warnings.simplefilter("always")
        got = fit_for_grid_many(db, pairs)
    assert got.keys() == one.keys()
    for p in pairs:
        assert (got[p] is None and one[p] is None) or _same(got[p], one[p])
    assert [str(x.message) for x in w_many] == [str(x.message) for x in w_one]


def _random_lists(seed):
    from paper_2002_06790_b200.model import OpSignature, ProfileRecord

    rng = np.random.default_rng(seed)
    lists = []
    for t in range(120):
        k = int(rng.integers(1, 5))
        n = int(rng.integers(1, 40))
        names = [f"f{j}" for j in range(k)]
        x = rng.uniform(-1e3, 1e3, (n, k)) * 10.0 ** rng.integers(-6, 7, k)
        style = t % 6
        if style == 1 and k > 1:
            x[:, 1] = 2.0 * x[:, 0]  # collinear
        elif style == 2:
            x[:, 0] = 7.0  # constant column (collinear with the intercept)
        elif style == 3:
            x = np.round(x)  # integer grid (duplicates likely for small n)
        coef = rng.normal(0, 3, k)
        y = np.abs(x @ coef + rng.uniform(1, 100)) + rng.uniform(1e-3, 1.0, n)
        if style == 4:
            y[:] = 5.0  # constant duration (ss_tot == 0)
        elif style == 5:
            y = y * 10.0 ** rng.integers(-9, 9)
        lists.append([ProfileRecord(OpSignature("Op", "hw", tuple(zip(names, map(float, row)))), float(v))
                      for row, v in zip(x.tolist(), y.tolist())])
    # an empty list, a list that mixes feature names, one that mixes op types
    lists.append([])
    lists.append(lists[0][:2] + [ProfileRecord(OpSignature("Op", "hw", (("zz", 1.0),)), 1.0)])
    lists.append(lists[0][:2] + [ProfileRecord(OpSignature("Other", "hw", lists[0][0].signature.arg_features), 1.0)])
    return lists


@pytest.mark.parametrize("seed", range(6))
def test_random_grids(seed):
    from paper_2002_06790_b200.lowering import fit_linear_many

    lists = _random_lists(seed)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        many = fit_linear_many(lists)
        for recs, m in zip(lists, many):
            assert _same(m, _per_list(recs)), recs[:2]


def test_without_the_stacked_gufunc(monkeypatch):
    """The per-matrix lstsq fallback (a numpy without the private gufunc) gives the same fits."""
    import paper_2002_06790_b200.lowering as L

    class NoGufunc:
        pass

    lists = _random_lists(7)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        want = [_per_list(r) for r in lists]
        monkeypatch.setattr(L.np.linalg, "_umath_linalg", NoGufunc(), raising=False)
        got = L.fit_linear_many(lists)
    assert all(_same(a, b) for a, b in zip(got, want))
