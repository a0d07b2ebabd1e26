"""Config-scale goldens from the UNMODIFIED reference (oracle/_ref, scalar table).

    python tests/golden/make_scale_golden.py c2    # full C2: 1e5 shots, seed 1 (~35 min on 8 cores)
    python tests/golden/make_scale_golden.py c3    # full C3: 1e6 shots, run_branch budget 65536 (~3 min)
    python tests/golden/make_scale_golden.py c45   # 64 C4 shot ids + 8 C5 shot ids (~5 min)

Writes tests/golden/scale_<part>.json (+ the full C2 values as raw little-endian
u16, gzip'd). The reference paths: run_naive (exec_naive.cpp:131-161) for C2,
run_branch (exec_branch.cpp:175-295) for C3, run_single_shot per id
(exec_naive.cpp:88-129) for C4/C5. The values hash is sha256 over the u64
little-endian per-shot values, so GPU tests compare whole runs bit for bit.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Reference  # noqa: E402
from paper_2308_03399_b200 import circuits as cc  # noqa: E402

OUT = Path(__file__).resolve().parent

C4_IDS = list(range(32)) + [313 * i + 17 for i in range(31)] + [9_999]
C5_IDS = [0, 1, 2, 3, 1234, 5000, 7777, 9_999]


def values_sha256(vals) -> str:
    return hashlib.sha256(np.ascontiguousarray(vals, dtype="<u8").tobytes()).hexdigest()


def counts_of(vals):
    u, c = np.unique(np.asarray(vals, dtype=np.uint64), return_counts=True)
    return {str(int(k)): int(n) for k, n in zip(u, c)}


def meta(cfg):
    t, nz = cfg["circuit"](), cfg["noise"]()
    return t, nz, {"circuit_sha256": hashlib.sha256(t.encode()).hexdigest(),
                   "noise_sha256": hashlib.sha256(nz.encode()).hexdigest(), "seed": cfg["seed"]}


def part_c2(ref):
    cfg = cc.CONFIGS["C2"]
    t, nz, m = meta(cfg)
    t0 = time.time()
    vals, st = ref.run(t, nz, "naive", cfg["shots"], cfg["seed"], workers=8)
    secs = time.time() - t0
    assert int(vals.max()) < 1 << 16
    (OUT / "scale_c2_values.u16.gz").write_bytes(gzip.compress(vals.astype("<u2").tobytes(), 9))
    m.update(shots=cfg["shots"], values_sha256=values_sha256(vals), checksum=hex(st.counts_checksum),
             num_keys=st.num_keys, seconds=secs, strategy="naive (scalar table), 8 workers",
             values_file="scale_c2_values.u16.gz")
    (OUT / "scale_c2.json").write_text(json.dumps(m, indent=1))
    print("C2", secs, "s", hex(st.counts_checksum))


def part_c3(ref):
    cfg = cc.CONFIGS["C3"]
    t, nz, m = meta(cfg)
    t0 = time.time()
    vals, st = ref.run(t, nz, "branch", cfg["shots"], cfg["seed"], workers=8, budget=65536)
    secs = time.time() - t0
    m.update(shots=cfg["shots"], budget=65536, values_sha256=values_sha256(vals), checksum=hex(st.counts_checksum),
             num_keys=st.num_keys, peak_states=st.peak_states, passes=st.passes, seconds=secs,
             counts=counts_of(vals), strategy="branch (scalar table), 8 workers")
    (OUT / "scale_c3.json").write_text(json.dumps(m, indent=1))
    print("C3", secs, "s", hex(st.counts_checksum), st.peak_states, st.passes)


def part_c45(ref):
    res = {}
    for key, ids in (("C4", C4_IDS), ("C5", C5_IDS)):
        cfg = cc.CONFIGS[key]
        t, nz, m = meta(cfg)
        v, secs = ref.run_ids(t, nz, ids, cfg["seed"], workers=8)
        m.update(ids=ids, values=[int(x) for x in v], seconds=secs)
        res[key] = m
        print(key, secs, "s")
    (OUT / "scale_c45.json").write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    ref = Reference()
    ref.select_kernels("scalar")
    for part in sys.argv[1:]:
        {"c2": part_c2, "c3": part_c3, "c45": part_c45}[part](ref)
