"""Generates tests/golden/*.json from the UNMODIFIED reference library
(oracle/_ref, compiled from /root/reference/proj/src by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures travel with the repo, so GPU-box tests compare against the
reference's own outputs without /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Reference  # noqa: E402
from paper_2308_03399_b200 import circuits as cc  # noqa: E402

OUT = Path(__file__).resolve().parent


def checksum(vals, width, has_measure=True):
    counts = {}
    for v in vals:
        k = format(int(v), "b").zfill(width) if has_measure else ""
        counts[k] = counts.get(k, 0) + 1
    h = 0xCBF29CE484222325
    for k in sorted(counts):
        for ch in (k + "=" + str(counts[k]) + ";").encode():
            h = ((h ^ ch) * 0x100000001B3) & ((1 << 64) - 1)
    return h, len(counts)


def main():
    ref = Reference()
    ref.select_kernels("scalar")

    # --- RNG known answers (Random123 KATs + the reference's uniform()) ---
    kat = {
        "philox": [
            {"ctr": [0, 0, 0, 0], "key": [0, 0]},
            {"ctr": [0xFFFFFFFF] * 4, "key": [0xFFFFFFFF] * 2},
            {"ctr": [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], "key": [0xA4093822, 0x299F31D0]},
        ],
        "uniform": [],
    }
    for e in kat["philox"]:
        e["out"] = ref.philox(e["ctr"], e["key"])
    for seed, shot, event in [(7, 0, 0), (7, 0, 3), (7, 1, 0), (7, 1, 3), (7, 12345, 0), (7, 12345, 3),
                              (1, 0, 1440), (0, 2**40 + 3, 2**33 + 1), (2**63 + 5, 99, 7)]:
        kat["uniform"].append({"seed": seed, "shot": shot, "event": event,
                               "u": ref.uniform(seed, shot, event).hex()})
    (OUT / "rng_kat.json").write_text(json.dumps(kat, indent=1))

    # --- C1 full run (1000 shots, seed 1) ---
    t, nz = cc.ghz(10), cc.depolarizing_model(0.01)
    vals, st = ref.run(t, nz, "naive", 1000, 1)
    bvals, bst = ref.run(t, nz, "batch", 1000, 1)
    assert (vals == bvals).all()
    (OUT / "c1_ghz10.json").write_text(json.dumps({
        "circuit": t, "noise": nz, "shots": 1000, "seed": 1, "values": [int(v) for v in vals],
        "checksum": hex(st.counts_checksum), "num_keys": st.num_keys, "batch_dispatches": bst.dispatch_count,
    }))

    # --- random mixed programs (cross-strategy recipe) ---
    rng = cc.SplitMix64(99)
    progs = []
    for rep in range(24):
        circ = cc.random_mixed(rng)
        noise = cc.depolarizing_model(0.08, as_kraus=(rep % 3 == 2))
        seed = 500 + rep
        v, _ = ref.run(circ, noise, "naive", 96, seed)
        branch = {}
        for budget in (1, 3, 64):
            bv, bs = ref.run(circ, noise, "branch", 96, seed, budget=budget)
            assert (bv == v).all()
            branch[str(budget)] = {"peak_states": bs.peak_states, "passes": bs.passes}
        progs.append({"circuit": circ, "noise": noise, "seed": seed, "shots": 96,
                      "values": [int(x) for x in v], "branch": branch})
    (OUT / "random_programs.json").write_text(json.dumps(progs))

    # --- dyn12 branch statistics ---
    t, nz = cc.dynamic(12), cc.depolarizing_model(0.01)
    dyn = {"circuit": t, "noise": nz, "shots": 4000, "seed": 1, "budgets": {}}
    for budget in (1, 64, 65536):
        v, s = ref.run(t, nz, "branch", 4000, 1, workers=8, budget=budget)
        dyn["budgets"][str(budget)] = {"peak_states": s.peak_states, "passes": s.passes,
                                       "checksum": hex(s.counts_checksum)}
    dyn["values"] = [int(x) for x in v]
    (OUT / "dyn12_branch.json").write_text(json.dumps(dyn))

    # --- per-shot samples of the large configs (sub-sampled by shot id) ---
    samples = {}
    for key, ids in (("C2", list(range(24)) + [99_999]), ("C4", [0, 1, 9_999]), ("C5", [0])):
        cfg = cc.CONFIGS[key]
        t, nz = cfg["circuit"](), cfg["noise"]()
        v, secs = ref.run_ids(t, nz, ids, cfg["seed"], workers=8)
        samples[key] = {"ids": ids, "values": [int(x) for x in v], "seed": cfg["seed"], "seconds": secs,
                        "circuit_sha256": hashlib.sha256(t.encode()).hexdigest(),
                        "noise_sha256": hashlib.sha256(nz.encode()).hexdigest()}
        print(key, "sample", secs, "s")
    (OUT / "config_samples.json").write_text(json.dumps(samples, indent=1))

    # --- instrumented-program dumps (lowering parity) ---
    dumps = {}
    for key, cfg in cc.CONFIGS.items():
        t, nz = cfg["circuit"](), cfg["noise"]()
        dumps[key] = hashlib.sha256(ref.program_dump(t, nz).encode()).hexdigest()
    t, nz = cc.qft(4), cc.depolarizing_model(0.05, True)
    dumps["qft4_kraus"] = hashlib.sha256(ref.program_dump(t, nz).encode()).hexdigest()
    (OUT / "program_dumps.json").write_text(json.dumps(dumps, indent=1))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
