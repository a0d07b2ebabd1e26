"""CPU model of the warp-parallel exact sequential scan (engine/exact_scan.cuh,
mirrored statement by statement with 32 numpy "lanes"): it must reproduce the
reference's sequential cumulative fl(cum + p) (statevector.cpp:185-197) bit
for bit — every running sum in full-scan mode (branch leaf tables) and the
first crossing / pick_outcome fallback in pick mode — including dyadic inputs
that force exact ties and binade changes."""
import math

import numpy as np

def seq(p, u):
    S=0.0; out=[]
    for x in p:
        S = S + x; out.append(S)
    return out
def frexp_e(S): return math.frexp(S)[1]
def warp_scan(p, u, record):
    count=len(p); S=0.0; last_nz=-1; res=None
    for c0 in range(0, count, 32):
        m = np.arange(c0, c0+32)
        pl = np.array([p[i] if i < count else 0.0 for i in m])
        nz = pl > 0
        if nz.any(): last_nz = c0 + int(np.nonzero(nz)[0].max())
        start=0
        while start < 32:
            if not (S >= 2.0**-1022):
                if S == 0.0:
                    nzl = [l for l in range(start,32) if nz[l]]
                    if not nzl:
                        for l in range(start,32):
                            if m[l] < count: record[m[l]] = 0.0
                        break
                    b = nzl[0]
                    for l in range(start,b):
                        if m[l] < count: record[m[l]] = 0.0
                else:
                    b = start
                Sn = S + pl[b]
                if c0+b < count: record[c0+b] = Sn
                if u < Sn and c0+b < count: return ('cross', c0+b)
                S = Sn; start = b+1; continue
            if not any(nz[l] for l in range(start,32)):
                # only zeros left in this chunk: S stays
                for l in range(start,32):
                    if m[l] < count: record[m[l]] = S
                break
            e = frexp_e(S); w = math.ldexp(1.0, e-53); a0 = int(S/w)
            k = [0]*32; bad=[False]*32
            for l in range(start,32):
                x = pl[l]/w
                if x >= 2.0**42: bad[l]=True
                else:
                    bad[l] = (x - math.floor(x)) == 0.5
                    k[l] = int(np.rint(x))
            pre = np.cumsum(k)
            a = a0 + pre
            brk = [l>=start and (bad[l] or a[l] >= 2**53) for l in range(32)]
            B = brk.index(True) if any(brk) else 32
            Sl = [float(a[l])*w for l in range(32)]
            for l in range(start,B):
                if m[l] < count: record[m[l]] = Sl[l]
            cross = [l for l in range(start,B) if m[l]<count and u < Sl[l]]
            if cross: return ('cross', c0+cross[0])
            if B > start: S = Sl[B-1]
            if B == 32: break
            Sn = S + pl[B]
            if m[B] < count: record[m[B]] = Sn
            if u < Sn and c0+B < count: return ('cross', c0+B)
            S = Sn; start = B+1
    return ('fallback', last_nz)


def _pick(p, u):
    cum, last = 0.0, -1
    for i, x in enumerate(p):
        cum += x
        if u < cum:
            return ("cross", i)
        if x > 0:
            last = i
    return ("fallback", last)


def test_full_scan_matches_sequential_sums():
    rng = np.random.default_rng(1)
    for trial in range(200):
        n = int(rng.integers(1, 11))
        a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        if trial % 3 == 0:
            a[rng.random(a.size) < 0.7] = 0
        if trial % 5 == 0:
            a[:int(rng.integers(0, a.size))] = 0
        if np.linalg.norm(a) > 0:
            a /= np.linalg.norm(a)
        p = [float(x.real * x.real + x.imag * x.imag) for x in a]
        rec = [None] * len(p)
        warp_scan(p, float("inf"), rec)
        assert rec == seq(p, 0)


def test_pick_matches_pick_outcome():
    rng = np.random.default_rng(2)
    for trial in range(1500):
        n = int(rng.integers(1, 9))
        a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        if trial % 3 == 0:
            a[rng.random(a.size) < 0.7] = 0
        if np.linalg.norm(a) > 0:
            a /= np.linalg.norm(a)
        if trial % 7 == 0:
            a *= 0.9  # sums below 1: fallback cases
        p = [float(x.real * x.real + x.imag * x.imag) for x in a]
        u = float(rng.random())
        assert warp_scan(p, u, [None] * len(p)) == _pick(p, u)


def test_dyadic_ties_and_binades():
    rng = np.random.default_rng(3)
    for _ in range(1000):
        p = [float(rng.integers(0, 8)) * 2.0 ** -int(rng.integers(1, 60)) for _ in range(1 << int(rng.integers(2, 8)))]
        u = float(rng.random()) * sum(p) * 1.1
        want = _pick(p, u)
        got = warp_scan(p, u, [None] * len(p))
        if want[0] == "cross":
            assert got == want
        rec = [None] * len(p)
        warp_scan(p, float("inf"), rec)
        assert rec == seq(p, 0)

