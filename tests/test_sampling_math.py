"""CPU check of the exactness argument behind the device terminal sampler
(sample_exact_kernel, kernels.cuh): advancing the reference's SEQUENTIAL fl
sum S_m = fl(S_{m-1} + p_m) over a chunk by one integer reduction
w * (a + sum(rint(p/w))) — valid when no p/w is a tie and the sum stays in
S's binade — gives exactly the sequential result (statevector.cpp:185-197).
Pure Python floats are IEEE binary64 with round-to-nearest-even."""

import math
import random

import pytest

CHUNK = 2048


def advance_exact(S, ps):
    """The kernel's exact-advance rule; None when it must replay serially."""
    if S < 2.0 ** -1022:
        return None
    _, e = math.frexp(S)                      # S in [2^(e-1), 2^e)
    w = math.ldexp(1.0, e - 53)
    a = int(S / w)
    D = 0
    for p in ps:
        x = p / w
        if x >= 2.0 ** 42 or x - math.floor(x) == 0.5:
            return None
        D += int(round(x))  # rint (no ties reach here)
    if a + D >= 2 ** 53:
        return None
    return (a + D) * w


def sequential(S, ps):
    for p in ps:
        S = S + p
    return S


@pytest.mark.parametrize("n,seed", [(14, 1), (16, 2), (18, 3)])
def test_integer_advance_equals_sequential_sum(n, seed):
    rng = random.Random(seed)
    # Porter-Thomas-like probabilities (random state), normalised in fl.
    amps = [complex(rng.gauss(0, 1), rng.gauss(0, 1)) for _ in range(1 << n)]
    norm = math.fsum(abs(a) ** 2 for a in amps)
    ps = [(a.real / math.sqrt(norm)) ** 2 + (a.imag / math.sqrt(norm)) ** 2 for a in amps]
    S_seq, S_adv = 0.0, 0.0
    advanced = serial = 0
    for c0 in range(0, len(ps), CHUNK):
        chunk = ps[c0:c0 + CHUNK]
        S_seq = sequential(S_seq, chunk)
        nxt = advance_exact(S_adv, chunk)
        if nxt is None:
            S_adv = sequential(S_adv, chunk)  # serial replay
            serial += 1
        else:
            S_adv = nxt
            advanced += 1
        assert S_adv == S_seq                 # bit-identical after every chunk
    if n >= 16:  # p/w ties get rarer with n (~2^-(n-1) per element): most chunks advance
        assert advanced > serial


def test_tie_is_detected():
    S = 0.5  # binade [0.5, 1): w = 2^-53
    w = 2.0 ** -53
    assert advance_exact(S, [1.5 * w]) is None     # exact half-ulp: parity-dependent
    assert advance_exact(S, [1.25 * w]) == S + w   # rint(1.25) = 1, like fl(S + 1.25w)
    assert sequential(S, [1.25 * w]) == S + w
