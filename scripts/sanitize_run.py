"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): resident (one-warp and CTA builds),
shot-branching, streamed exact tile passes (JIT + interpreter), Kraus decide
steps, measure / reset specials, the fused-matrix passes (FMA and MMA builds)
and the exact sampler. Not a benchmark."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc  # noqa: E402

eng = Engine(0)
cases = [
    ("C1 resident-warp", cc.ghz(10), cc.depolarizing_model(0.01), "batch", 64, {}),
    ("C1 branch", cc.ghz(10), cc.depolarizing_model(0.01), "branch", 64, {}),
    ("dyn12 resident-cta", cc.dynamic(12, rounds=2), cc.depolarizing_model(0.02), "batch", 16, {}),
    ("dyn12 branch", cc.dynamic(12, rounds=2), cc.depolarizing_model(0.02), "branch", 64, {"branch_budget": 16}),
    ("qv14 exact jit", cc.quantum_volume(14, depth=2, seed=1), cc.qv_noise(), "batch", 4, {}),
    ("qv14 exact interp", cc.quantum_volume(14, depth=2, seed=1), cc.qv_noise(), "batch", 4, {"interpret_only": True}),
    ("qv14 fused fma", cc.quantum_volume(14, depth=2, seed=1), cc.qv_noise(), "batch", 4, {"fused_matrices": True}),
    ("qv14 fused fma 12-qubit tiles", cc.quantum_volume(14, depth=2, seed=1), cc.qv_noise(), "batch", 4,
     {"fused_matrices": True, "tile_qubits": 12}),
    ("qv12 fused many shots (128-thread sampler CTAs)", cc.quantum_volume(12, depth=2, seed=1), cc.qv_noise(),
     "batch", 1200, {"fused_matrices": True, "resident_max_qubits": 1}),
    ("rnd13 kraus streamed", cc.random_layers(13, depth=2, seed=3), cc.thermal_noise(0.05, 0.1), "batch", 4,
     {"resident_max_qubits": 1, "tile_qubits": 11}),
    ("rnd14 kraus streamed epilogue (several tiles per CTA)", cc.random_layers(14, depth=2, seed=4),
     cc.thermal_noise(0.05, 0.1), "batch", 256, {"resident_max_qubits": 1, "tile_qubits": 10}),
    ("dyn12 streamed specials", cc.dynamic(12, rounds=1), cc.depolarizing_model(0.02), "batch", 4,
     {"resident_max_qubits": 1, "tile_qubits": 10}),
]
only = sys.argv[1] if len(sys.argv) > 1 else ""
for name, circ, noise, mode, shots, kw in cases:
    if only and only not in name:
        continue
    prog = Program.from_text(circ, noise)
    run = eng.run_branch if mode == "branch" else eng.run_batch
    r = run(prog, RunOptions(shots=shots, seed=3, **kw))
    print(name, "ok", r.dispatch_count, flush=True)
if not only or "epilogue" in only:  # the opt-in Kraus-site epilogue, several tiles per CTA
    os.environ["SHOTSIM_B200_EPILOGUE"] = "1"
    prog = Program.from_text(cc.random_layers(14, depth=2, seed=4), cc.thermal_noise(0.05, 0.1))
    r = eng.run_batch(prog, RunOptions(shots=256, seed=3, resident_max_qubits=1, tile_qubits=10))
    os.environ["SHOTSIM_B200_EPILOGUE"] = "0"
    print("rnd14 kraus epilogue on ok", r.dispatch_count, flush=True)
if not only or "jit" in only:  # the per-pass NVRTC-specialised fused kernels (11- and 12-qubit tiles)
    os.environ["SHOTSIM_B200_FUSED_JIT"] = "1"
    for tile in (11, 12):
        prog = Program.from_text(cc.quantum_volume(14, depth=2, seed=1), cc.qv_noise())
        r = eng.run_batch(prog, RunOptions(shots=4, seed=3, fused_matrices=True, tile_qubits=tile))
        assert r.specialised_shapes == r.fused_passes
        print("qv14 fused jit tile", tile, "ok", r.dispatch_count, flush=True)
    os.environ["SHOTSIM_B200_FUSED_JIT"] = "0"
if not only or "mma" in only:
    os.environ["SHOTSIM_B200_FUSED_MMA"] = "1"
    prog = Program.from_text(cc.quantum_volume(14, depth=2, seed=1), cc.qv_noise())
    r = eng.run_batch(prog, RunOptions(shots=4, seed=3, fused_matrices=True))
    print("qv14 fused mma ok", r.dispatch_count, flush=True)
