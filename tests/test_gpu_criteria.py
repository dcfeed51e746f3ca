"""Reference acceptance properties on the device path: the Schur-block estimator is
unbiased (reference `tests/test_skeleton.py:131-147`, criterion 3), and the adaptive loop's
skeletons are the one-shot LUPP prefix of the concatenated blocks (`test_skeleton.py:221-232`,
criterion 2)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def rs():
    import paper_2310_09417_b200 as rs

    return rs


@pytest.mark.parametrize("kind", ["gaussian", "srtt", "sparsesign"])
def test_estimator_unbiased_within_standard_errors(rs, kind):
    a, _ = rs.gen_fast_decay(100, 100, 1e-16, rs.RngStream(20))
    spec = rs.SketchSpec(kind, n=100, ell=20)
    state = rs.adaptive_init(a, 20, spec, rs.RngStream(21))
    w = rs.interpolation_matrix(state)
    truth = np.linalg.norm(a - w @ a[state.perm[:20]]) ** 2
    draws = np.empty(300)
    for i in range(draws.size):
        e, _ = rs.adaptive_step(state, a, spec, rs.RngStream(5000).child(i))
        draws[i] = e ** 2
    se = draws.std(ddof=1) / np.sqrt(draws.size)
    assert abs(draws.mean() - truth) <= 5 * se


def test_adaptive_equals_one_shot_prefix(rs):
    from paper_2310_09417_b200 import _device
    from paper_2310_09417_b200.lu_state import _draw_block

    a, _ = rs.gen_fast_decay(120, 100, 1e-16, rs.RngStream(31))
    spec = rs.SketchSpec("gaussian", n=100, ell=100)
    res = rs.rand_lupp_adaptive(a, b=10, tau=1e-6 * np.linalg.norm(a), spec=spec, rng=rs.RngStream(32))
    A = _device.as_matrix(a)
    blocks = [_draw_block(A, spec, rs.RngStream(32).child(t), 10).cpu().numpy() for t in range(res.rank // 10)]
    one = rs.lupp(np.hstack(blocks))
    assert np.array_equal(res.row_idx, one.perm[: res.rank])
