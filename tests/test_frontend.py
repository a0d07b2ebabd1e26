"""CPU: the product's host front-end (circuit text / noise JSON / instrument)
lowers every config bit-identically to the reference's instrument()."""

import hashlib

import pytest

from conftest import golden
from paper_2308_03399_b200 import ConfigError, Program, circuits as cc
from paper_2308_03399_b200.api import bitstring, counts_checksum_of_values, counts_from_values


@pytest.mark.parametrize("key", list(cc.CONFIGS))
def test_lowering_matches_reference_dump(key):
    cfg = cc.CONFIGS[key]
    dump = Program.from_text(cfg["circuit"](), cfg["noise"]()).dump()
    assert hashlib.sha256(dump.encode()).hexdigest() == golden("program_dumps.json")[key]


def test_kraus_lowering_matches_reference_dump():
    dump = Program.from_text(cc.qft(4), cc.depolarizing_model(0.05, True)).dump()
    assert hashlib.sha256(dump.encode()).hexdigest() == golden("program_dumps.json")["qft4_kraus"]


def test_event_and_site_census():
    # C2 1424 gates + 1424 Pauli sites, 1440 events; C3 116 events.
    p = Program.from_text(cc.quantum_volume(16), cc.qv_noise())
    ops = p.ops()
    assert sum(o.kind == 0 for o in ops) == 1424 and sum(o.kind == 1 for o in ops) == 1424
    assert p.num_events == 1440 and p.sampling_eligible
    d = Program.from_text(cc.dynamic(12), cc.depolarizing_model(0.01))
    assert d.num_events == 116 and not d.sampling_eligible
    k = Program.from_text(cc.random_layers(20), cc.thermal_noise())
    assert sum(o.kind == 2 for o in k.ops()) == 590


def test_sampling_eligibility_rules():
    # conditional read of a terminal clbit disables sampling (program.cpp:105-119)
    c = cc.CircuitText(2, 2).op("h", [0]).op("x", [1], cond=(1, 1)).op("measure", [0], clbits=[0])
    assert not Program.from_text(c.text()).sampling_eligible
    c = cc.CircuitText(2, 2).op("h", [0]).op("measure", [0], clbits=[0]).op("x", [1])
    assert not Program.from_text(c.text()).sampling_eligible
    assert Program.from_text(cc.ghz(3)).sampling_eligible


def test_invalid_circuits_raise_like_the_reference():
    with pytest.raises(ValueError):
        Program.from_text("qubits 1\nclbits 1\nmeasure q0 -> c5\n")
    with pytest.raises(ValueError):
        Program.from_text("qubits 2\ncx q0,q0\n")
    with pytest.raises(ConfigError):
        Program.from_text("qubits 1\nfoo q0\n")
    with pytest.raises(ConfigError):
        Program.from_text(cc.ghz(2), '{"rules":[{"gates":["h"],"arity":1,"channel":{"type":"pauli",'
                                     '"terms":[[0.5,"I"],[0.4,"X"]]}}]}')
    with pytest.raises(ConfigError):  # completeness violated
        Program.from_text(cc.ghz(2), '{"rules":[{"gates":["h"],"arity":1,"channel":{"type":"kraus",'
                                     '"matrices":[[[1,0],[0,0],[0,0],[0.5,0]]]}}]}')


def test_results_folding():
    assert bitstring(5, 4) == "0101"
    assert counts_from_values([1, 1, 2], 2, True) == {"01": 2, "10": 1}
    assert counts_from_values([0, 0], 0, False) == {"": 2}
    g = golden("c1_ghz10.json")
    cs, keys = counts_checksum_of_values(g["values"], 10, True)
    assert hex(cs) == g["checksum"] and keys == g["num_keys"]
