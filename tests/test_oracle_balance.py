"""Pins for oracle/balance.py -- Eq. (3), Eq. (4)."""
import numpy as np
import pytest

from oracle import balance as ob


def test_ibd_worked_values():
    assert ob.ibd([2, 2, 2, 2]) == 0.0
    assert ob.ibd([1, 3, 8, 4]) == 2.0                  # avg 4, (3+1+4+0)/4
    assert ob.ibd([0, 16]) == 8.0                       # exactly at threshold: not "exceeds" (Q24)
    with pytest.raises(ValueError):
        ob.ibd([])


def test_ibd_permutation_invariant_and_zero_iff_equal():
    rng = np.random.default_rng(0)
    for _ in range(50):
        x = rng.integers(0, 50, size=int(rng.integers(1, 40)))
        assert ob.ibd(x) == pytest.approx(ob.ibd(rng.permutation(x)), rel=1e-12, abs=0)
        assert (ob.ibd(x) == 0.0) == bool(np.all(x == x[0]))


def test_eq4_worked_value():
    # A800, FeatureDim 128, 4 blocks: Load = WB = 8*128*4*4 / 1935e9, MMA = 8*15*128 / 156e12
    load = 16384 / 1935e9
    mma = 15360 / 156e12
    assert ob.eq4_time("A800", 128, 4) == pytest.approx(2 * load + mma, rel=1e-12)
    assert ob.eq4_time("A800", 128, 4) == pytest.approx(1.7033e-8, rel=1e-4)


def test_eq4_linearity_and_monotonicity():
    rng = np.random.default_rng(1)
    for _ in range(1000):
        p = ["RTX4090", "A800", "H100"][int(rng.integers(0, 3))]
        fd, tb = int(rng.integers(1, 1024)), int(rng.integers(1, 64))
        t = ob.eq4_time(p, fd, tb)
        assert ob.eq4_time(p, fd, tb + 1) > t and ob.eq4_time(p, fd + 1, tb) > t
        mma = ob.eq4_time(p, fd, 0)
        assert ob.eq4_time(p, fd, 2 * tb) - mma == pytest.approx(2 * (t - mma), rel=1e-9)


def _powerlaw_rwo(rng, W):
    nb = np.minimum((rng.pareto(1.2, W) * 3).astype(np.int64), 400)
    nb[rng.random(W) < 0.1] = 0
    return np.concatenate([[0], np.cumsum(nb)])


@pytest.mark.parametrize("seed", range(20))
@pytest.mark.parametrize("cap", [32, 100])
@pytest.mark.parametrize("precision", ["tf32", "fp16"])
def test_schedule_coverage_and_cap(seed, cap, precision):
    rng = np.random.default_rng(seed)
    rwo = _powerlaw_rwo(rng, int(rng.integers(1, 500)))
    units = ob.build_units(rwo, cap, True, precision)
    ob.check_coverage(units, rwo)
    wb = ob.wb_cost(precision)
    for (w0, nw, b0, b1, split, seg, nseg, slot) in units:
        assert b1 - b0 <= cap and nw <= ob.WMAX
        if split == ob.NO_SPLIT:
            cost = sum(int(rwo[w + 1] - rwo[w]) + wb for w in range(w0, w0 + nw))
            assert nw == 1 or cost <= cap + wb
        else:
            assert nseg == -(-int(rwo[w0 + 1] - rwo[w0]) // cap) and 0 <= seg < nseg
    # identity schedule: one unit per window, one write-back each
    ident = ob.build_units(rwo, cap, False, precision)
    assert len(ident) == rwo.size - 1
    ob.check_coverage(ident, rwo)


@pytest.mark.parametrize("seed", range(20))
def test_balanced_max_over_mean_not_worse(seed):
    """S:575 acceptance 6: balanced max/mean predicted time <= identity schedule's on power-law plans."""
    rng = np.random.default_rng(100 + seed)
    rwo = _powerlaw_rwo(rng, 300)
    nonempty = [(w, 1, int(rwo[w]), int(rwo[w + 1]), 0, 0, 1, 0) for w in range(rwo.size - 1)
                if rwo[w + 1] > rwo[w]]
    bal = [u for u in ob.build_units(rwo, 32, True) if u[3] > u[2]]
    assert ob.mean_ratio(ob.unit_times(bal, rwo)) <= ob.mean_ratio(ob.unit_times(nonempty, rwo))


def test_split_segments_even():
    rwo = np.array([0, 100])
    units = ob.build_units(rwo, 32, True)
    assert [(u[2], u[3]) for u in units] == [(0, 25), (25, 50), (50, 75), (75, 100)]
    assert [u[7] for u in units] == [0, 1, 2, 3]


def test_auto_cap():
    assert ob.auto_cap(0) == 32 and ob.auto_cap(10) == 32
    assert ob.auto_cap(14_000_000) == 512   # ceil(14e6 / 28416) = 493 -> 512
    assert ob.auto_cap(10 ** 10) == 4096


@pytest.mark.parametrize("seed", range(20))
@pytest.mark.parametrize("cap", [32, 100])
@pytest.mark.parametrize("precision", ["tf32", "fp16"])
def test_grouped_schedule_keeps_windows_whole(seed, cap, precision):
    """Reading R7b (balance AUTO, IBD <= 8): whole windows only -- no unit splits a window,
    every window appears in exactly one unit in order, groups respect the concatenation rule
    (cost <= cap + wb unless a unit is a single window, at most WMAX windows), and a unit is
    closed only when the next window would break that rule (greedy maximality)."""
    rng = np.random.default_rng(300 + seed)
    rwo = _powerlaw_rwo(rng, int(rng.integers(1, 500)))
    units = ob.build_units(rwo, cap, False, precision, group=True)
    ob.check_coverage(units, rwo)
    wb = ob.wb_cost(precision)
    nb = np.diff(rwo)
    for k, (w0, nw, b0, b1, split, seg, nseg, slot) in enumerate(units):
        assert split == ob.NO_SPLIT and nseg == 1 and b0 == rwo[w0] and b1 == rwo[w0 + nw]
        cost = int(sum(nb[w0:w0 + nw])) + wb * nw
        assert nw <= ob.WMAX and (nw == 1 or cost <= cap + wb)
        nxt = w0 + nw
        if k + 1 < len(units) and nb[w0:w0 + nw].max(initial=0) <= cap and nb[nxt] <= cap:
            assert nw == ob.WMAX or cost + int(nb[nxt]) + wb > cap + wb
    # with no window above the cap, grouping equals the balanced schedule (nothing to split)
    small = np.concatenate([[0], np.cumsum(np.minimum(nb, cap))])
    assert ob.build_units(small, cap, False, precision, group=True) == ob.build_units(small, cap, True, precision)


# Paper-literal schedule, written out by hand (TC blocks redistributed so that
# TBs take "nearly uniform computation time", "a maximum threshold of 32 TC blocks per TB";
# the split of a long window is even and its segments are reduced by the cross-row
# write-back of P:404; short windows are concatenated, reading R7 / SURVEY Q16).
# Blocks per window: 3, 70, 5, 40, 2, 1, 30, 64, 0, 4 -> rwo below.  IBD by hand: avg 21.9,
# |dev| = 18.9+48.1+16.9+18.1+19.9+20.9+8.1+42.1+21.9+17.9 = 232.8 -> 23.28 > 8.
# Units (w0, nw, b0, b1, split_id, seg, nseg, slot), cap 32, TF32 (C write-back = 1 block):
#   w0 (3 blocks) alone: the next window is split;
#   w1 (70 > 32) -> ceil(70/32) = 3 even segments at 3 + floor(70k/3): [3,26) [26,49) [49,73);
#   w2 (5) alone; w3 (40) -> 2 segments [78,98) [98,118);
#   w4 + w5 (2+1 blocks, cost (2+1)+(1+1) = 5 <= 33); w6 (30) would make 5+31 = 36 > 33 -> alone;
#   w7 (64) -> 2 segments [151,183) [183,215); w8 (empty) + w9 (4): cost 1+5 = 6.
HAND_RWO = [0, 3, 73, 78, 118, 120, 121, 151, 215, 215, 219]
NS = ob.NO_SPLIT
HAND_UNITS = [
    (0, 1, 0, 3, NS, 0, 1, 0),
    (1, 1, 3, 26, 0, 0, 3, 0), (1, 1, 26, 49, 0, 1, 3, 1), (1, 1, 49, 73, 0, 2, 3, 2),
    (2, 1, 73, 78, NS, 0, 1, 0),
    (3, 1, 78, 98, 1, 0, 2, 3), (3, 1, 98, 118, 1, 1, 2, 4),
    (4, 2, 118, 121, NS, 0, 1, 0),
    (6, 1, 121, 151, NS, 0, 1, 0),
    (7, 1, 151, 183, 2, 0, 2, 5), (7, 1, 183, 215, 2, 1, 2, 6),
    (8, 2, 215, 219, NS, 0, 1, 0),
]


def test_paper_literal_cap32_schedule_by_hand():
    blocks = np.diff(HAND_RWO)
    assert ob.ibd(blocks) == pytest.approx(23.28, abs=1e-12)
    units = ob.build_units(HAND_RWO, ob.PAPER_CAP, True, "tf32")
    assert units == HAND_UNITS
    assert max(b1 - b0 for (_, _, b0, b1, *_r) in units) <= 32
