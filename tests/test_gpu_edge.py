"""Reference edge cases on the device, through the operator-level ABI with
explicit draws (the *_with hooks, exec_batch.hpp:57-62) and hand-written
(unnormalised) segments:

* pick_outcome strictness / fallback / degenerate table
  (tests/test_statevector.cpp:210-221, statevector.cpp:185-197);
* the batch measure's rounding-slack fallback (exec_batch.cpp:169-182);
* the Kraus fallback to the last matrix with its own probability
  (exec_naive.cpp:29-42 / exec_batch.cpp:98-118);
* DegenerateDistribution from measure and from terminal sampling.
"""

import numpy as np
import pytest

from paper_2308_03399_b200 import BatchState, Program, RunOptions
from paper_2308_03399_b200._lib import DegenerateDistribution, ShotsimError

pytestmark = pytest.mark.gpu

MEAS1 = "qubits 1\nclbits 1\nx q0\nmeasure q0 -> c0\n"


def _measure_with(engine, amps, u):
    """The measure op (1 qubit, the reference's only measure arity) applied
    with draw u to a segment set to amps (possibly unnormalised)."""
    prog = Program.from_text(MEAS1)
    mi = next(i for i, o in enumerate(prog.ops()) if o.kind == 3)
    b = BatchState(engine, prog, [0], 0)
    b.write_segment(0, np.asarray(amps, dtype=np.complex128))
    b.apply_op(mi, [u])
    return int(b.cregs()[0]), b.segments()[0]


# test_statevector.cpp:210-221 restated over the two outcomes of a 1-qubit
# measure (p_0 = |0.5|^2 = 0.25 exactly).
@pytest.mark.parametrize("amps,u,want", [
    ([0.5, 0.75 ** 0.5], 0.0, 0),            # u = 0 picks the first nonzero outcome
    ([0.5, 0.75 ** 0.5], 0.25, 1),           # strict: u == cum moves on
    ([0.5, 0.75 ** 0.5], 0.2499, 0),
    ([0.0, 1.0], 0.0, 1),                    # zero-probability outcome unreachable
    ([0.5 + 0.5j, 0.5 + 0.5j], 0.999999, 1),
])
def test_pick_outcome_strictness(engine, amps, u, want):
    m, seg = _measure_with(engine, amps, u)
    assert m == want
    assert np.count_nonzero(seg) == 1 and abs(abs(seg[want]) - 1.0) < 1e-15


def test_pick_outcome_slack_fallback(engine):
    """Probabilities sum below 1 and u lies above the sum: the last outcome with
    p > 0 (pick_outcome fallback; the batch measure's slack dispatch,
    exec_batch.cpp:169-182)."""
    m, seg = _measure_with(engine, [0.5, np.sqrt(0.4999999)], 0.9999999999)
    assert m == 1
    m, _ = _measure_with(engine, [np.sqrt(0.4999999), 0.0], 0.99999999999)
    assert m == 0  # skips the zero tail


def test_measure_degenerate(engine):
    with pytest.raises(DegenerateDistribution):
        _measure_with(engine, [0.0, 0.0], 0.5)


def test_terminal_sampling_degenerate(engine):
    prog = Program.from_text("qubits 2\nclbits 2\nmeasure q0 -> c0\nmeasure q1 -> c1\n")
    b = BatchState(engine, prog, [0], 0)
    b.write_segment(0, np.zeros(4, dtype=np.complex128))
    with pytest.raises(DegenerateDistribution):
        b.run()


AD = ('{"rules":[{"gates":["id"],"arity":1,"channel":{"type":"kraus","matrices":'
      '[[[1,0],[0,0],[0,0],[0.5,0]],[[0,0],[0.8660254037844386,0],[0,0],[0,0]]]}}]}')


def test_kraus_last_matrix_fallback(engine):
    """State of norm^2 = 0.5: the Kraus probabilities sum to 0.5; a draw above
    it selects the LAST matrix scaled by its own 1/sqrt(p)."""
    prog = Program.from_text("qubits 1\nclbits 0\nid q0\n", AD)
    ki = next(i for i, o in enumerate(prog.ops()) if o.kind == 2)
    a = np.array([0.5, 0.5j], dtype=np.complex128)  # |a|^2 = 0.5
    m0 = np.array([[1, 0], [0, 0.5]])
    m1 = np.array([[0, 0.8660254037844386], [0, 0]])
    p0 = np.linalg.norm(m0 @ a) ** 2
    p1 = np.linalg.norm(m1 @ a) ** 2
    for u, sel, p in ((0.2, m0, p0), (p0 + 0.01, m1, p1), (0.9, m1, p1)):
        b = BatchState(engine, prog, [0], 0)
        b.write_segment(0, a)
        b.apply_op(ki, [u])
        got = b.segments()[0]
        want = (sel @ a) / np.sqrt(p)
        assert np.allclose(got, want, rtol=0, atol=1e-15), (u, got, want)


def _with_gate_matrix(prog, op_index, entries):
    """A copy of `prog` whose gate op `op_index` carries `entries` (2x2,
    row-major complex) — through ssb_program_from_flat, the flat ABI."""
    import ctypes as C
    from paper_2308_03399_b200 import _lib
    f = prog.flat()
    mats = np.ctypeslib.as_array(f.matrices, shape=(f.num_matrices * _lib.MATRIX_STRIDE,)).copy()
    slot = f.ops[op_index].matrix
    for e, v in enumerate(entries):
        mats[slot * _lib.MATRIX_STRIDE + 2 * e] = complex(v).real
        mats[slot * _lib.MATRIX_STRIDE + 2 * e + 1] = complex(v).imag
    g = _lib.FlatProgram.from_buffer_copy(f)
    g.matrices = mats.ctypes.data_as(_lib._pd)
    h = C.c_void_p()
    _lib.check(_lib.load().ssb_program_from_flat(C.byref(g), C.byref(h)))
    return Program(h.value)


def test_norm_check_accepts_and_rejects(engine):
    """check_norms (exec_batch.cpp:217-224): a clean run passes with values
    identical to the fused executor's; an op that breaks the norm (a
    non-unitary gate matrix, only expressible through the flat ABI) fails
    the run with the reference's runtime_error."""
    from paper_2308_03399_b200 import circuits as cc
    prog = Program.from_text(cc.qft(5), cc.depolarizing_model(0.05, as_kraus=True))
    clean = engine.run_batch(prog, RunOptions(shots=64, seed=3, record_shot_values=True))
    checked = engine.run_batch(prog, RunOptions(shots=64, seed=3, record_shot_values=True, check_norms=True))
    assert (checked.shot_values == clean.shot_values).all()
    base = Program.from_text("qubits 2\nclbits 2\nx q0\nid q0\nmeasure q0 -> c0\nmeasure q1 -> c1\n")
    bad = _with_gate_matrix(base, 1, [1, 0, 0, 1.5])
    engine.run_batch(bad, RunOptions(shots=8, seed=1))  # unchecked: runs
    with pytest.raises(ShotsimError, match="norm drifted after op 1"):
        engine.run_batch(bad, RunOptions(shots=8, seed=1, check_norms=True))
