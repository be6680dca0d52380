"""The closed form behind shuffle_resolve_kernel (shuffle.cuh), checked exhaustively on small
cases against the sequential Fisher-Yates loop of the oracle (shuffle.py:100-134 semantics:
z[i] <-> z[J[i]] for i = n-1 .. lim).  Pure host code; no device."""

import itertools
import random


def sequential(z, J, lim):
    z = list(z)
    for i in range(len(z) - 1, lim - 1, -1):
        z[i], z[J[i]] = z[J[i]], z[i]
    return z


def closed_form(z0, J, lim):
    n = len(z0)
    steps = {}
    for i in range(lim, n):
        steps.setdefault(J[i], []).append(i)

    def ns(i):
        later = [m for m in steps.get(J[i], []) if m > i]
        return min(later) if later else None

    def F(x):
        while True:
            later = [m for m in steps.get(x, []) if m > x]
            if not later:
                return x
            x = min(later)

    out = []
    for i in range(n):
        if i >= lim:
            a = ns(i)
            out.append(z0[F(a)] if a is not None else z0[J[i]])
        else:
            out.append(z0[F(i)])
    return out


def test_closed_form_exhaustive_small():
    for n in range(1, 7):
        for J in itertools.product(*[range(i + 1) for i in range(n)]):
            for lim in range(0, n + 1):
                assert closed_form(list(range(n)), J, lim) == sequential(range(n), J, lim), (n, J, lim)


def test_closed_form_random():
    rng = random.Random(7)
    for _ in range(2000):
        n = rng.randrange(1, 200)
        lim = rng.choice((1, 1, 0, rng.randrange(0, n + 1)))
        J = [rng.randrange(i + 1) for i in range(n)]
        assert closed_form(list(range(n)), J, lim) == sequential(range(n), J, lim)
