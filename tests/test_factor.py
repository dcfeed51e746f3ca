"""The `factor` path (`harness.factor_run`, `cli.cmd_factor`) against the reference's
own output files (tests/golden/make_factor_golden.py)."""
import os
import types

import numpy as np
import pytest

from paper_2310_09417_b200 import factor as fx
from paper_2310_09417_b200.skeleton import TraceRecord

GOLD = os.path.join(os.path.dirname(__file__), "golden", "factor")
CASES = ("rel", "abs_cap")


def _meta(name):
    with open(os.path.join(GOLD, name + ".meta.txt")) as fh:
        kv = dict(item.split("=", 1) for item in fh.read().split())
    return kv


def _read_gold(name):
    m = _meta(name)
    a = np.load(os.path.join(GOLD, "a.npy"))
    k = int(m["rank"])
    idx = np.loadtxt(os.path.join(GOLD, name + ".indices.txt"), dtype=np.int64).reshape(-1)
    w = np.fromfile(os.path.join(GOLD, name + ".w.f64"), dtype="<f8").reshape((a.shape[0], k), order="F")
    trace = []
    with open(os.path.join(GOLD, name + ".trace.csv")) as fh:
        lines = fh.read().splitlines()[2:]
    for ln in lines:
        kk, e, nu, mu = ln.split(",")
        trace.append(TraceRecord(int(kk), float(e), float(nu) if nu else None, float(mu) if mu else None))
    return a, m, idx, w, trace


def _same_bytes(p, q):
    with open(p, "rb") as f1, open(q, "rb") as f2:
        return f1.read() == f2.read()


@pytest.mark.parametrize("name", CASES)
def test_writers_match_reference_bytes(tmp_path, name):
    _, m, idx, w, trace = _read_gold(name)
    res = types.SimpleNamespace(row_idx=idx, w=w, trace=trace, status=m["status"], rank=int(m["rank"]))
    prefix = str(tmp_path / name)
    code = fx.write_factor_outputs(prefix, res)
    assert code == (fx.EXIT_OK if m["status"] == "ok" else fx.EXIT_NOT_CONVERGED)
    for ext in (".indices.txt", ".w.f64", ".trace.csv"):
        assert _same_bytes(prefix + ext, os.path.join(GOLD, name + ext)), ext


def test_trace_writer_optional_estimates(tmp_path):
    res = types.SimpleNamespace(row_idx=np.array([3, 1]), w=np.eye(2), status="rank_exhausted",
                                trace=[TraceRecord(2, 0.5, 0.25, 0.125)])
    assert fx.write_factor_outputs(str(tmp_path / "x"), res) == fx.EXIT_RANK_EXHAUSTED
    body = (tmp_path / "x.trace.csv").read_text().splitlines()
    assert body == ["# randskel-trace v1", "k,e_schur,est_norm_ur,est_max_ur", "2,0.5,0.25,0.125"]


def test_cli_usage_errors(tmp_path, capsys):
    raw = tmp_path / "a.f64"
    np.arange(6, dtype="<f8").tofile(raw)
    assert fx.main(["--input", str(raw)]) == fx.EXIT_USAGE
    assert fx.main(["--input", str(raw), "--shape", "4,4"]) == fx.EXIT_USAGE
    assert fx.main(["--input", str(tmp_path / "missing.npy")]) == fx.EXIT_USAGE


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_factor_run_matches_reference(tmp_path, name):
    a, m, idx, w, trace = _read_gold(name)
    cfg = fx.FactorConfig(b=int(m["b"]), tau=float(m["tau"]), relative=m["relative"] == "True",
                          seed=int(m["seed"]), max_rank=None if m["max_rank"] == "None" else int(m["max_rank"]))
    tau_abs = fx.resolve_tau(a, cfg)
    assert abs(tau_abs - float(m["tau_abs"])) <= 1e-12 * float(m["tau_abs"])
    res = fx.factor_run(a, cfg)
    assert res.rank == int(m["rank"]) and res.status == m["status"]
    np.testing.assert_array_equal(np.asarray(res.row_idx), idx)
    na = np.linalg.norm(a)
    assert [r.k for r in res.trace] == [r.k for r in trace]
    assert max(abs(r.e_schur - g.e_schur) for r, g in zip(res.trace, trace)) <= 1e-12 * na
    prefix = str(tmp_path / name)
    code = fx.write_factor_outputs(prefix, res)
    assert code == (fx.EXIT_OK if m["status"] == "ok" else fx.EXIT_NOT_CONVERGED)
    assert _same_bytes(prefix + ".indices.txt", os.path.join(GOLD, name + ".indices.txt"))
    w_ours = np.fromfile(prefix + ".w.f64", dtype="<f8").reshape(w.shape, order="F")
    r_ours = np.linalg.norm(a - w_ours @ a[idx]) / na
    r_ref = np.linalg.norm(a - w @ a[idx]) / na
    assert r_ours <= 1.5 * r_ref + 1e-13


@pytest.mark.gpu
def test_factor_cli_end_to_end(tmp_path):
    a = np.load(os.path.join(GOLD, "a.npy"))
    raw = tmp_path / "a.f64"
    a.ravel(order="F").astype("<f8").tofile(raw)
    m = _meta("rel")
    out = str(tmp_path / "f")
    code = fx.main(["--input", str(raw), "--shape", f"{a.shape[0]},{a.shape[1]}", "--b", m["b"],
                    "--tau", m["tau"], "--relative", "--seed", m["seed"], "--out", out])
    assert code == fx.EXIT_OK
    assert _same_bytes(out + ".indices.txt", os.path.join(GOLD, "rel.indices.txt"))
