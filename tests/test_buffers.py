"""The result-buffer text form (reference buffers.py:8-21, 129-200).

Fixtures are the reference's own `serialize` output (tests/golden/
make_golden.py --buffers-only): parsing them with `load_buffer` and writing
them back with `dump_buffer` reproduces the reference's bytes exactly; the
GPU test runs the same batch through the B200 pool and compares the parsed
results with the reference's within the 1e-10 bar."""

import json
from pathlib import Path

import pytest

import paper_2406_03466_b200 as qv

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_buffers.json"


@pytest.fixture(scope="module")
def golden_buffers():
    if not GOLDEN.exists():
        pytest.skip("golden_buffers.json missing; run tests/golden/make_golden.py --buffers-only")
    return json.loads(GOLDEN.read_text())


def test_reference_text_round_trips_exactly(golden_buffers):
    for case in golden_buffers:
        buf = qv.load_buffer(case["text"])
        assert qv.dump_buffer(buf) == case["text"]
        assert qv.serialize is qv.dump_buffer and qv.deserialize is qv.load_buffer


def test_parsed_values_are_exact(golden_buffers):
    buf = qv.load_buffer(golden_buffers[0]["text"])
    assert buf.metadata == {"a.b-c_d": -7, "label": "run 1", "ok": True, "scale": 0.1 + 0.2, "vqpu_count": 4}
    assert buf.child("k0+").expectation == 1.0 / 3.0
    assert buf.child("with space").expectation == -2.5e-17
    assert buf.child("c").counts == {"000": 2, "011": 1, "101": 5} and buf.child("c").shots == 8
    assert buf.child("d").distribution == {"000": 0.1, "001": 0.1 + 0.2, "111": 0.6}


@pytest.mark.parametrize("text,err", [
    ("nope\nnqubits 2\n", "header"),
    ("qvirt-buffer v1\n", "nqubits"),
    ("qvirt-buffer v1\nnqubits 2\nchild a\nmeta k 1\n", "meta after"),
    ("qvirt-buffer v1\nnqubits 2\nexpectation 1.0\n", "before any child"),
    ("qvirt-buffer v1\nnqubits 2\nchild a\nprob 00 0.5\nprob 00 0.5\n", "duplicate prob"),
    ("qvirt-buffer v1\nnqubits 2\nchild a\nshots 2\ncount 01 1\ncount 01 1\n", "duplicate count"),
    ("qvirt-buffer v1\nnqubits 2\nmeta k 1\nmeta k 2\n", "duplicate meta"),
    ("qvirt-buffer v1\nnqubits 2\nchild a\nbogus 1\n", "unrecognized"),
    ("qvirt-buffer v1\nnqubits 2\nchild a\nprob 00 0.4\n", "sum"),
])
def test_malformed_text_is_rejected(text, err):
    with pytest.raises(ValueError, match=err):
        qv.load_buffer(text)


def test_dump_rejects_bad_metadata():
    buf = qv.ResultBuffer(n_qubits=1, metadata={"bad key": 1})
    with pytest.raises(ValueError, match="metadata key"):
        qv.dump_buffer(buf)
    with pytest.raises(ValueError, match="scalar"):
        qv.dump_buffer(qv.ResultBuffer(n_qubits=1, metadata={"k": [1]}))


@pytest.mark.gpu
def test_b200_pool_output_matches_reference_dump(gpu, golden_buffers):
    case = golden_buffers[1]
    batch = []
    for c in case["batch"]:
        circ = qv.Circuit(case["n"], tuple(qv.Gate(qv.GateKind(k), tuple(t), a) for k, t, a in c["gates"]),
                          name=c["name"])
        obs = c["observable"]
        if obs is not None:
            terms = [qv.PauliTerm(tuple(tuple(f) for f in factors), coef) for factors, coef in obs["terms"]]
            circ = circ.with_observable(terms[0] if obs["constant"] is None else qv.Observable(tuple(terms),
                                                                                                 obs["constant"]))
        batch.append(circ)
    buf = qv.ResultBuffer(n_qubits=case["n"])
    qv.execute_parallel(buf, batch, qv.VqpuPoolConfig(n_virtual_qpus=case["n_virtual_qpus"]))
    got, want = qv.load_buffer(qv.dump_buffer(buf)), qv.load_buffer(case["text"])
    assert got.metadata == want.metadata
    for a, b in zip(got.children, want.children, strict=True):
        assert a.name == b.name
        if b.expectation is not None:
            assert a.expectation == pytest.approx(b.expectation, abs=1e-10)
        if b.distribution is not None:
            keys = set(a.distribution) | set(b.distribution)
            assert max(abs(a.distribution.get(k, 0.0) - b.distribution.get(k, 0.0)) for k in keys) < 1e-10
