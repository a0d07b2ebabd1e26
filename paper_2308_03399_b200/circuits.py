"""Synthetic workloads of BASELINE.json in the reference's
lossless circuit text format (circuit_io.cpp:53-77) plus noise-model JSON
(noise.cpp:328-365). Reproducible with a self-specified splitmix64 stream, so
the GPU engine and the reference CPU oracle read byte-identical inputs.

  C1 ghz(10)              + depolarizing(0.01)           1000 shots, seed 1
  C2 quantum_volume(16)   + depolarizing 1% + readout    1e5 shots  (headline)
  C3 dynamic(12)          + depolarizing(0.01)           1e6 shots  (branching)
  C4 random_layers(20)    + thermal relaxation (Kraus)   1e4 shots
  C5 quantum_volume(24)   + depolarizing 1%              1e4 shots
"""

from __future__ import annotations

import json
import math
from typing import List, Optional, Sequence, Tuple

MASK64 = (1 << 64) - 1


class SplitMix64:
    def __init__(self, seed: int):
        self.x = seed & MASK64

    def next(self) -> int:
        self.x = (self.x + 0x9E3779B97F4A7C15) & MASK64
        z = self.x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next() >> 11) * (2.0 ** -53)

    def below(self, n: int) -> int:
        return self.next() % n

    def shuffle(self, items: List) -> None:  # Fisher-Yates
        for i in range(len(items) - 1, 0, -1):
            j = self.below(i + 1)
            items[i], items[j] = items[j], items[i]


def g17(v: float) -> str:
    return "%.17g" % v


class CircuitText:
    """Builder for the reference circuit text format."""

    def __init__(self, num_qubits: int, num_clbits: int = 0):
        self.n = num_qubits
        self.c = num_clbits
        self.lines: List[str] = []

    def op(self, name: str, qubits: Sequence[int] = (), params: Sequence[float] = (),
           clbits: Sequence[int] = (), cond: Optional[Tuple[int, int]] = None) -> "CircuitText":
        s = name
        if qubits:
            s += " " + ",".join(f"q{q}" for q in qubits)
        if params:
            s += " " + ",".join(g17(p) for p in params)
        if clbits:
            s += " -> " + ",".join(f"c{c}" for c in clbits)
        if cond is not None:
            s += f" if {cond[0]}=={cond[1]}"
        self.lines.append(s)
        return self

    def measure_all(self) -> "CircuitText":
        self.c = max(self.c, self.n)
        for q in range(self.n):
            self.op("measure", [q], clbits=[q])
        return self

    def text(self) -> str:
        return f"qubits {self.n}\nclbits {self.c}\n" + "".join(l + "\n" for l in self.lines)


# ---- noise models -------------------------------------------------------------
def depolarizing_model(rate: float, as_kraus: bool = False) -> str:
    """make_depolarizing_model (noise.cpp:375-392) — evaluated by each engine."""
    return json.dumps({"model": "depolarizing", "rate": rate, "as_kraus": as_kraus})


ONE_Q = ["x", "y", "z", "h", "s", "sdg", "t", "tdg", "p", "u"]
TWO_Q = ["cx", "cp", "swap"]


def _depol_terms(p: float, k: int):
    strings = 4 ** k
    each = p / strings
    ident = 1.0 - each * (strings - 1)
    letters = "IXYZ"
    out = [[ident, "I" * k]]
    for code in range(1, strings):
        out.append([each, "".join(letters[(code >> (2 * s)) & 3] for s in range(k))])
    return out


def qv_noise(rate: float = 0.01, readout: Optional[float] = 0.01) -> str:
    """C2/C5: depolarizing on 1q (not id) and 2q gates; readout flip on id."""
    rules = [
        {"gates": ONE_Q, "arity": 1, "channel": {"type": "pauli", "terms": _depol_terms(rate, 1)}},
        {"gates": TWO_Q, "arity": 2, "channel": {"type": "pauli", "terms": _depol_terms(rate, 2)}},
    ]
    if readout:
        rules.append({"gates": ["id"], "arity": 1,
                      "channel": {"type": "pauli", "terms": [[1.0 - readout, "I"], [readout, "X"]]}})
    return json.dumps({"rules": rules})


def thermal_noise(gamma: float = 0.005, lam: float = 0.01) -> str:
    """C4: thermal relaxation as Kraus — 3 matrices on u, the
    9-matrix tensor product on cx (slot 0 = low matrix axis)."""
    a = math.sqrt(1 - gamma) * math.sqrt(1 - lam)
    g = math.sqrt(gamma)
    b = math.sqrt(1 - gamma) * math.sqrt(lam)
    k1 = [[[1, 0], [0, 0], [0, 0], [a, 0]], [[0, 0], [g, 0], [0, 0], [0, 0]], [[0, 0], [0, 0], [0, 0], [b, 0]]]

    def kron(hi, lo):  # (hi ⊗ lo)[r1 r0, c1 c0] = hi[r1,c1] * lo[r0,c0]
        out = []
        for r in range(4):
            for c in range(4):
                x = hi[(r >> 1) * 2 + (c >> 1)][0] * lo[(r & 1) * 2 + (c & 1)][0]
                out.append([x, 0.0])
        return out

    k2 = [kron(h, l) for h in k1 for l in k1]
    return json.dumps({"rules": [
        {"gates": ["u"], "arity": 1, "channel": {"type": "kraus", "matrices": k1}},
        {"gates": ["cx"], "arity": 2, "channel": {"type": "kraus", "matrices": k2}},
    ]})


# ---- circuits -------------------------------------------------------------------
def ghz(n: int = 10) -> str:
    c = CircuitText(n)
    c.op("h", [0])
    for i in range(1, n):
        c.op("cx", [i - 1, i])
    return c.measure_all().text()


def qft(n: int, measure: bool = True) -> str:
    """qft_circuit (circuit.cpp:106-123)."""
    c = CircuitText(n)
    for k in range(n - 1, -1, -1):
        c.op("h", [k])
        for j in range(k):
            c.op("cp", [j, k], [math.pi / float(1 << (k - j))])
    for j in range(n // 2):
        c.op("swap", [j, n - 1 - j])
    return c.measure_all().text() if measure else c.text()


def _angle(rng: SplitMix64) -> float:
    return rng.uniform() * 2.0 * math.pi - math.pi


def quantum_volume(n: int = 16, depth: Optional[int] = None, seed: int = 2308, readout_ids: bool = True) -> str:
    """QV: per layer a seeded pairing, each pair an SU(4) block
    `u x; u y; 3x[cx x,y; u x; u y]`; then `id` on every qubit; measure_all."""
    rng = SplitMix64(seed)
    depth = n if depth is None else depth
    c = CircuitText(n)
    for _ in range(depth):
        perm = list(range(n))
        rng.shuffle(perm)
        for b in range(n // 2):
            x, y = perm[2 * b], perm[2 * b + 1]
            c.op("u", [x], [_angle(rng), _angle(rng), _angle(rng)])
            c.op("u", [y], [_angle(rng), _angle(rng), _angle(rng)])
            for _ in range(3):
                c.op("cx", [x, y])
                c.op("u", [x], [_angle(rng), _angle(rng), _angle(rng)])
                c.op("u", [y], [_angle(rng), _angle(rng), _angle(rng)])
    if readout_ids:
        for q in range(n):
            c.op("id", [q])
    return c.measure_all().text()


def dynamic(n: int = 12, rounds: int = 4) -> str:
    """C3 dyn12: each round H on all, CX ladder, measure q_r -> c_r, reset q_r,
    x q_{r+4} if (1<<r)==(1<<r); then measure_all."""
    c = CircuitText(n, n)
    for r in range(rounds):
        for q in range(n):
            c.op("h", [q])
        for q in range(n - 1):
            c.op("cx", [q, q + 1])
        c.op("measure", [r], clbits=[r])
        c.op("reset", [r])
        c.op("x", [(r + 4) % n], cond=(1 << r, 1 << r))
    return c.measure_all().text()


def random_layers(n: int = 20, depth: int = 20, seed: int = 2020) -> str:
    """C4 rnd20: per layer random u on every qubit, then CX brickwork offset d%2."""
    rng = SplitMix64(seed)
    c = CircuitText(n)
    for d in range(depth):
        for q in range(n):
            c.op("u", [q], [_angle(rng), _angle(rng), _angle(rng)])
        for q in range(d % 2, n - 1, 2):
            c.op("cx", [q, q + 1])
    return c.measure_all().text()


def random_mixed(rng: SplitMix64, max_qubits: int = 4) -> str:
    """Random programs mixing gates, measures, resets, conditionals and
    barriers — the recipe of test_cross_strategy.cpp:17-60."""
    n = 1 + rng.below(max_qubits)
    c = CircuitText(n, n)
    length = 4 + rng.below(12)
    for _ in range(length):
        q = rng.below(n)
        kind = rng.below(12)
        if kind in (0, 1):
            c.op("h", [q])
        elif kind == 2:
            c.op("x", [q])
        elif kind == 3:
            c.op("p", [q], [rng.uniform() * 6.0 - 3.0])
        elif kind == 4:
            if n >= 2:
                q2 = rng.below(n)
                if q2 == q:
                    q2 = (q2 + 1) % n
                c.op("cx", [q, q2])
        elif kind == 5:
            c.op("measure", [q], clbits=[q])
        elif kind == 6:
            c.op("reset", [q])
        elif kind == 7:
            mask = 1 << rng.below(n)
            c.op("x", [q], cond=(mask, mask if rng.below(2) else 0))
        elif kind == 8:
            c.lines.append("barrier")
        elif kind == 9:
            if n >= 2:
                q2 = (q + 1 + rng.below(n - 1)) % n
                c.op("cp", [q, q2], [rng.uniform() * 6.0 - 3.0])
        elif kind == 10:
            c.op("u", [q], [_angle(rng), _angle(rng), _angle(rng)])
        else:
            c.op("s", [q])
    if rng.below(2):
        c.measure_all()
    return c.text()


def random_bursts(rng: SplitMix64, n: int = 12, bursts: int = 24, clbits: int = 4) -> str:
    """Streamed-path stress circuits: bursts of every gate kind on random
    qubit pairs (so segments of many kinds form inside each tile pass), a few
    conditionals on pre-measured clbits, then measure_all."""
    c = CircuitText(n, max(n, clbits))
    for b in range(clbits):
        c.op("h", [b])
        c.op("measure", [b], clbits=[b])
    one = ["id", "x", "y", "z", "h", "s", "sdg", "t", "tdg"]
    for _ in range(bursts):
        a = rng.below(n)
        b = (a + 1 + rng.below(n - 1)) % n
        for _ in range(2 + rng.below(10)):
            q = a if rng.below(2) else b
            kind = rng.below(16)
            cond = None
            if rng.below(10) == 0:
                m = 1 << rng.below(clbits)
                cond = (m, m if rng.below(2) else 0)
            if kind < 5:
                c.op("u", [q], [_angle(rng), _angle(rng), _angle(rng)], cond=cond)
            elif kind < 8:
                c.op(one[rng.below(len(one))], [q], cond=cond)
            elif kind == 8:
                c.op("p", [q], [_angle(rng)], cond=cond)
            elif kind < 12:
                c.op("cx", [q, b if q == a else a], cond=cond)
            elif kind < 14:
                c.op("cp", [a, b] if rng.below(2) else [b, a], [_angle(rng)], cond=cond)
            else:
                c.op("swap", [a, b], cond=cond)
    return c.measure_all().text()


CONFIGS = {
    "C1": dict(name="ghz10", circuit=lambda: ghz(10), noise=lambda: depolarizing_model(0.01), shots=1000, seed=1),
    "C2": dict(name="qv16", circuit=lambda: quantum_volume(16), noise=lambda: qv_noise(0.01, 0.01), shots=100_000,
               seed=1),
    "C3": dict(name="dyn12", circuit=lambda: dynamic(12), noise=lambda: depolarizing_model(0.01), shots=1_000_000,
               seed=1),
    "C4": dict(name="rnd20", circuit=lambda: random_layers(20), noise=lambda: thermal_noise(), shots=10_000, seed=1),
    "C5": dict(name="qv24", circuit=lambda: quantum_volume(24), noise=lambda: qv_noise(0.01, None), shots=10_000,
               seed=1),
}
