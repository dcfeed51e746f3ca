"""The divergence-analysis tool (tools/cfg2_divergence.py) replays the oracle's pivoting
exactly, so the near-tie it reports is the oracle's own."""
import importlib.util
import os

import numpy as np

import randskel_oracle as orc

_TOOL = os.path.join(os.path.dirname(__file__), "..", "tools", "cfg2_divergence.py")


def _tool():
    spec = importlib.util.spec_from_file_location("cfg2_divergence", _TOOL)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_eliminate_matches_oracle_lupp():
    tool = _tool()
    g = np.random.default_rng(7)
    for m, w in ((300, 64), (129, 17), (64, 64)):
        s = g.standard_normal((m, w)) * np.logspace(0, -9, w)
        A, order = tool.eliminate(s, w)
        L, U, perm, nc = orc.lupp(s)
        assert nc == w
        np.testing.assert_array_equal(order, perm)
        np.testing.assert_allclose(np.triu(A[:w]), U, rtol=0, atol=1e-13 * np.abs(U).max())


def test_candidates_rank_the_next_pivot_first():
    tool = _tool()
    g = np.random.default_rng(3)
    s = g.standard_normal((200, 8))
    rows = np.arange(1000, 1200)
    A, order = tool.eliminate(s, 3)
    v, ids, top = tool.candidates(A, order, 3, rows)
    _, _, perm, _ = orc.lupp(s)
    assert ids[top[0]] == rows[perm[3]]
