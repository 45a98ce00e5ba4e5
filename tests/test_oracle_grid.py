"""Pins for oracle/grid.py: SPEC.md simgrid worked examples and identities."""
import numpy as np
import pytest

from oracle.grid import Grid


def test_create_rejects_zero():
    with pytest.raises(ValueError):
        Grid(0)


def test_all_gather_examples():
    g = Grid(2)
    out = g.all_gather([np.array([1, 2]), np.array([3, 4])])
    assert all(np.array_equal(o, [1, 2, 3, 4]) for o in out)
    g1 = Grid(1)
    out = g1.all_gather([np.array([5.0])])
    assert np.array_equal(out[0], [5.0]) and g1.comm_log[0]["bytes"] == 0


def test_reduce_scatter_and_all_reduce_examples():
    g = Grid(2)
    out = g.reduce_scatter([np.array([1.0, 1.0]), np.array([2.0, 2.0])])
    assert np.array_equal(out[0], [3.0]) and np.array_equal(out[1], [3.0])
    out = g.all_reduce([np.array([1.0, 2.0]), np.array([10.0, 20.0])])
    assert all(np.array_equal(o, [11.0, 22.0]) for o in out)
    with pytest.raises(ValueError):
        g.reduce_scatter([np.ones(3), np.ones(3)])


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
def test_identities(p):
    rng = np.random.default_rng(p)
    g = Grid(p)
    xs = [rng.normal(size=(4 * p, 3)) for _ in range(p)]
    # AG o RS == AR
    ar = g.all_reduce(xs)
    agrs = g.all_gather(g.reduce_scatter(xs))
    for a, b in zip(ar, agrs):
        assert np.allclose(a, b, rtol=0, atol=1e-13)
    # dense single-buffer oracle: AR = direct elementwise sum
    assert np.allclose(ar[0], np.sum(np.stack(xs), axis=0))
    # A2A involution under axis swap
    ys = [rng.normal(size=(2 * p, 5, 3 * p)) for _ in range(p)]
    there = g.all_to_all(ys, split_axis=2, concat_axis=0)
    back = g.all_to_all(there, split_axis=0, concat_axis=2)
    for a, b in zip(ys, back):
        assert np.array_equal(a, b)
    # A2A by direct index bookkeeping: dst d, source src -> rows [src*2p..], cols of chunk d
    for d in range(p):
        for src in range(p):
            blk = there[d][src * 2 * p:(src + 1) * 2 * p]
            assert np.array_equal(blk, ys[src][:, :, d * 3:(d + 1) * 3])
    # ring pass: p passes reconstruct the identity
    z = [np.array([float(i)]) for i in range(p)]
    w = z
    for _ in range(p):
        w = g.ring_pass(w)
    assert all(np.array_equal(a, b) for a, b in zip(w, z))


def test_payload_convention_and_ledger():
    g = Grid(4)
    g.all_gather([np.zeros((2, 8))] * 4, bpe=2)       # full = 8x8x2 = 128 B -> 3/4 -> 96
    g.all_reduce([np.zeros(8)] * 4, bpe=4)            # 32 B x 2 x 3/4 = 48
    assert [e["bytes"] for e in g.comm_log] == [96, 48]
    hid = g.track(0, 100)
    g.release(hid)
    assert g.alloc[0] == 0 and g.peak[0] == 100
    with pytest.raises(ValueError):
        g.track(1, -5)
