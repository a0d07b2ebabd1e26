"""Generates tests/golden/density_exact.json from the UNMODIFIED reference's
exact density-matrix evolver (exact_creg_distribution / exact_distribution,
proj/src/density.cpp:280-306) through oracle/_ref (oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_density_golden.py
Cases follow the reference's own density tests (test_density.cpp:106-192) and
the statistical acceptance gate (acceptance_main.cpp:154-170), plus the
noise/op kinds the GPU evolver has kernels for (Pauli sites, Kraus channels
of 1 and 2 qubits incl. the 16-matrix depolarizing Kraus form, resets,
conditions, two intermediate measure sites) and the n = 10 maximum size.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Reference  # noqa: E402
from paper_2308_03399_b200 import circuits as cc  # noqa: E402

OUT = Path(__file__).resolve().parent / "density_exact.json"

FLIP_1PCT = lambda gate: json.dumps({"rules": [  # noqa: E731  (table_one(), test_density.cpp:113-133)
    {"gates": [gate], "arity": 1, "channel": {"type": "pauli", "terms": [[0.99, "I"], [0.01, "X"]]}}]})


def cases():
    depol = cc.depolarizing_model(0.01, False)
    out = []
    for n in range(2, 7):  # acceptance_main.cpp:156-158
        out.append(("qft%d_depol" % n, cc.qft(n), depol, None))
    out.append(("qft3_noiseless", cc.qft(3), "", [0, 1, 2]))
    out.append(("h_flip", "qubits 1\nclbits 1\nh q0\nmeasure q0 -> c0\n", FLIP_1PCT("h"), [0]))
    out.append(("x_flip", "qubits 1\nclbits 1\nx q0\nmeasure q0 -> c0\n", FLIP_1PCT("x"), [0]))
    out.append(("intermediate", "qubits 2\nclbits 2\nh q0\nmeasure q0 -> c0\nx q1 if 1==1\nmeasure q1 -> c1\n",
                "", None))
    out.append(("reset", "qubits 1\nclbits 1\nh q0\nreset q0\nmeasure q0 -> c0\n", "", None))
    out.append(("qft4_depol_kraus", cc.qft(4), cc.depolarizing_model(0.02, True), [3, 1]))
    out.append(("dyn6_depol", cc.dynamic(6, 2), cc.depolarizing_model(0.02, False), [5, 0, 2]))
    out.append(("rnd5_thermal", cc.random_layers(5, 4, 77), cc.thermal_noise(0.05, 0.1), [0, 4]))
    out.append(("ghz10_depol", cc.ghz(10), depol, [9, 0]))
    out.append(("qv8_readout", cc.quantum_volume(8, 3, 11), cc.qv_noise(0.02, 0.03), None))
    # A 2q channel longer than 16 matrices: the thermal tensor product with
    # every matrix split in two halves (18 matrices, still complete).
    rules = json.loads(cc.thermal_noise(0.05, 0.1))["rules"]
    h = 0.5 ** 0.5
    rules[1]["channel"]["matrices"] = [[[h * x, h * y] for x, y in m] for m in rules[1]["channel"]["matrices"] for _ in (0, 1)]
    out.append(("rnd4_kraus18", cc.random_layers(4, 3, 5), json.dumps({"rules": rules}), [1, 2]))
    # A 2q Pauli site longer than 16 terms: 5% depolarizing with four terms
    # listed twice at half weight (20 terms; duplicates are legal).
    labels = [a + b for a in "IXYZ" for b in "IXYZ"]
    terms = [[1 - 0.05 * 15 / 16 if l == "II" else 0.05 / 16, l] for l in labels]
    terms = [t for t in terms if t[1] not in ("XX", "YY", "ZZ", "XZ")] + \
            [[t[0] / 2, t[1]] for t in terms if t[1] in ("XX", "YY", "ZZ", "XZ") for _ in (0, 1)]
    pauli20 = json.dumps({"rules": [{"gates": ["cx"], "arity": 2, "channel": {"type": "pauli", "terms": terms}}]})
    out.append(("ghz5_pauli20", cc.ghz(5), pauli20, [0, 4]))
    return out


def main():
    ref = Reference()
    res = {"generator": "tests/golden/make_density_golden.py (reference exact_creg_distribution)", "cases": []}
    for name, circ, noise, qubits in cases():
        keys, probs = ref.exact_creg_distribution(circ, noise)
        entry = {"name": name, "circuit": circ, "noise": noise,
                 "keys": [int(k) for k in keys], "probs": [float(p) for p in probs]}
        if qubits is not None:
            entry["qubits"] = qubits
            entry["marginal"] = [float(x) for x in ref.exact_distribution(circ, noise, qubits)]
        res["cases"].append(entry)
        print(name, len(keys), "entries", flush=True)
    errors = []
    deep = "qubits 1\nclbits 1\n" + "h q0\nmeasure q0 -> c0\n" * 3 + "h q0\n"
    errors.append({"name": "three_intermediate", "circuit": deep, "noise": "", "error": "CapacityError"})
    errors.append({"name": "n11", "circuit": cc.ghz(11), "noise": "", "error": "CapacityError"})
    cond_meas = "qubits 2\nclbits 2\nh q0\nmeasure q0 -> c0\nmeasure q1 -> c1 if 1==1\nh q1\nmeasure q1 -> c1\n"
    errors.append({"name": "conditional_intermediate", "circuit": cond_meas, "noise": "", "error": "invalid_argument"})
    for e in errors:
        try:
            ref.exact_creg_distribution(e["circuit"], e["noise"])
            raise SystemExit(f"{e['name']}: reference did not raise")
        except RuntimeError as ex:
            assert e["error"] in str(ex), (e["name"], str(ex))
    res["errors"] = errors
    OUT.write_text(json.dumps(res, indent=1) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
