"""CPU property test of the window-independent argmin summary used by K1 (NearMin,
paper_2511_00796_b200/csrc/train.cu): keeping, for the bit patterns b0, b0+1, b0+2 above the
smallest per-step time, the first rank reaching each is enough to recover the reference's
argmin of cost = window * per_step (first rank of minimal cost, oracle/oracle.c:337) for
every window. Brute force with IEEE binary64 products (numpy) on adversarial near ties."""
import numpy as np
import pytest


def summary(x):
    bits = x.view(np.int64)
    b0 = bits.min()
    keys = []
    for i in range(3):
        hit = np.nonzero(bits == b0 + i)[0]
        keys.append(int(hit[0]) if hit.size else None)
    return b0, keys


def winner_from_summary(b0, keys, w):
    xs = np.array([b0, b0 + 1, b0 + 2], dtype=np.int64).view(np.float64)
    costs = np.float64(w) * xs
    c0 = costs[0]
    win = min(k for k, c in zip(keys, costs) if k is not None and c == c0)
    return win, c0


def brute(x, w):
    c = np.float64(w) * x
    m = c.min()
    return int(np.nonzero(c == m)[0][0]), m


@pytest.mark.parametrize("seed", range(6))
def test_summary_recovers_argmin_for_every_window(seed):
    rng = np.random.default_rng(seed)
    for trial in range(200):
        base = rng.uniform(1e-3, 1e3)
        n = int(rng.integers(1, 64))
        # per-step times clustered within a few ulps of each other, plus far-away ones
        off = rng.integers(0, 6, size=n)
        x = (np.full(n, base).view(np.int64) + off).view(np.float64)
        far = rng.random(n) < 0.3
        x[far] *= rng.uniform(1.0, 2.0, size=far.sum())
        b0, keys = summary(x)
        for w in list(range(1, 130)) + [255, 1000, 12345]:
            assert winner_from_summary(b0, keys, w) == brute(x, w), (trial, w)
