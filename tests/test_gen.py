"""Generator checks (CPU): exact edge counts, CSR invariants, determinism."""
import numpy as np
import pytest

import gen


def _check_csr(g):
    rp, ci = g.row_ptr, g.col_idx
    assert rp[0] == 0 and (np.diff(rp) >= 0).all() and rp[-1] == ci.size
    assert ci.min(initial=0) >= 0 and ci.max(initial=0) < g.n_src
    d = np.diff(ci.astype(np.int64))
    starts = np.zeros(ci.size, bool)
    starts[rp[:-1][rp[:-1] < ci.size]] = True
    assert (d[~starts[1:]] > 0).all(), "rows must be strictly ascending (no duplicate edges)"


def test_tiny_config():
    g = gen.make_graph("tiny")
    assert (g.n_dst, g.nnz) == (1024, 16384)
    assert list(g.degrees()[:3]) == [0, 1, 1024]
    _check_csr(g)
    assert np.array_equal(g.col_idx[g.row_ptr[2]:g.row_ptr[3]], np.arange(1024))


def test_determinism():
    a = gen.random_graph(500, 7000, 42)
    b = gen.random_graph(500, 7000, 42)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    c = gen.random_graph(500, 7000, 43)
    assert not np.array_equal(a.col_idx, c.col_idx)


def test_features_regimes():
    x = gen.features((1000,), 1, 0, gen.REAL)
    assert x.min() >= -1 and x.max() < 1
    assert np.array_equal(x * 2 ** 23, np.round(x * 2 ** 23))
    e = gen.features((1000,), 1, 1, gen.UNIT)
    assert e.min() >= 0 and e.max() < 1
    i = gen.features((1000,), 1, 2, gen.INT, lo=-8, hi=8)
    assert set(np.unique(i)) <= set(range(-8, 9)) and len(np.unique(i)) == 17


@pytest.mark.slow
def test_rand100k_exact_edges():
    """PAPER.md P:601 / Table tab:dataset P:618: 48.0M edges; exact under SURVEY L9."""
    g = gen.make_graph("rand100k")
    assert g.nnz == 48_000_000
    d = g.degrees()
    assert (d == 2000).sum() == 20000 and (d == 100).sum() == 80000
    _check_csr(g)


def test_lognormal_exact_sum_and_shape():
    d = gen.degrees_lognormal(232965 // 10, 114615892 // 10, 1.2, 21657, 7)
    assert d.sum() == 114615892 // 10 and d.min() >= 1 and d.max() <= 21657


def test_to_bf16_round_to_nearest_even():
    """gen.to_bf16 equals torch's fp32 -> bfloat16 conversion (RNE), and the
    decoded values are exactly the bf16 values."""
    import torch
    x = gen.features((4096, 7), 5, 0) * np.float32(37.0)
    x = np.concatenate([x.ravel(), np.float32([0.0, -0.0, 1.0, 1.00390625, 1.01171875, 3.0e38, -2.5e-38])])
    bits, dec = gen.to_bf16(x)
    t = torch.from_numpy(x).to(torch.bfloat16)
    assert np.array_equal(bits, t.view(torch.int16).numpy().view(np.uint16))
    assert np.array_equal(dec, t.to(torch.float32).numpy())
