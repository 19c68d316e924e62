"""Circuit-file grammar, the CLI's host logic and exit codes (CPU), mirroring the reference's
pkg/tests/test_cli.py; the GPU-backed subcommands are in test_gpu_cli.py."""

from __future__ import annotations

import json

import pytest

import paper_1601_07195_b200 as sv
from paper_1601_07195_b200.circuitfile import parse_circuit_text
from paper_1601_07195_b200.cli import check_memory, classify_failure, main

BELL = "qubits 2\nH 0\nCX 0 1\n"


def test_full_grammar():
    text = """
    # every construct in one file
    qubits 4
    H 0
    X 1
    Y 2
    Z 3
    RK 2 0        # phase pi/2
    CX 0 1
    CRK 3 1 2
    U 0  0.0 0.0 1.0 0.0 1.0 0.0 0.0 0.0
    CU 2 3  1.0 0.0 0.0 0.0 0.0 0.0 0.0 1.0
    """
    circ = parse_circuit_text(text)
    assert circ.n == 4 and circ.gate_count == 9
    assert [op.control for op in circ.gates] == [None, None, None, None, None, 0, 1, None, 2]
    assert [op.name for op in circ.gates] == ["H", "X", "Y", "Z", "R2", "CX", "CR3", "U", "CU"]
    assert (circ.gates[4].gate.mat == sv.phase_r(2).mat).all()
    assert (circ.gates[7].gate.mat == sv.pauli_x().mat).all()


@pytest.mark.parametrize("text,match", [
    ("H 0\nqubits 2\n", "qubits"), ("qubits 2\nH 0\nQQ 1\n", "line 3"), ("qubits 2\nCX 0\n", "line 2"),
    ("qubits 2\nU 0 1.0\n", "line 2"), ("qubits 2\nH 2\n", "line 2"), ("qubits 2\nCX 1 1\n", "line 2"),
    ("qubits 1\nU 0 2.0 0.0 0.0 0.0 0.0 0.0 2.0 0.0\n", "unitary"), ("qubits two\n", "line 1"),
    ("qubits 2\nRK x 0\n", "line 2"), ("qubits 2\nRK 0 0\n", "line 2"), ("", "line 1"), ("# only\n", "qubits"),
    ("qubits 0\n", "qubit count"), ("qubits 2\nU 0 a 0 0 0 0 0 0 0\n", "numbers"),
])
def test_parse_errors(text, match):
    with pytest.raises(sv.CircuitParseError, match=match):
        parse_circuit_text(text)


def test_exit_codes_without_a_gpu(tmp_path):
    bell = tmp_path / "bell.qc"
    bell.write_text(BELL)
    assert main(["run", str(bell), "--ranks", "3"]) == 2
    assert main(["run", str(bell), "--ranks", "8"]) == 2
    assert main(["run", str(tmp_path / "absent.qc")]) == 2
    assert main(["run", str(bell), "--transport", "tcp"]) == 2
    assert main(["run", str(bell), "--fusion", "7"]) == 2  # l_c > m
    bad = tmp_path / "bad.qc"
    bad.write_text("qubits 2\nH 9\n")
    assert main(["run", str(bad)]) == 3
    huge = tmp_path / "huge.qc"
    huge.write_text("qubits 44\nH 0\n")
    assert main(["run", str(huge)]) == 4
    assert main(["run"]) == 2 and main(["no-such-command"]) == 2


def test_failure_classification_and_memory_guard():
    assert classify_failure(sv.TransportError("down")) == 5
    wrapped = RuntimeError("rank 1 failed")
    wrapped.__cause__ = sv.TransportError("down")
    assert classify_failure(wrapped) == 5
    assert classify_failure(RuntimeError("other")) == 1
    assert classify_failure(sv.CircuitParseError(3, "x")) == 3
    check_memory(20, 0, False, 1 << 22)
    with pytest.raises(sv.ResourceError):
        check_memory(40, 0, False, 1 << 22)  # 17.6 TB
    check_memory(36, 3, False, 1 << 22)       # config 4: 128 GiB per GPU
    with pytest.raises(sv.ResourceError):
        check_memory(36, 3, True, 1 << 22)    # ... but not all eight slices on one GPU


def test_bounds_table(capsys):
    assert main(["bounds", "--m-range", "29:31", "--format", "json"]) == 0
    doc = json.loads(capsys.readouterr().out)
    assert doc["schema"] == 1 and [r["m"] for r in doc["rows"]] == [29, 30, 31]
    first = doc["rows"][0]
    # the reference's Table 2 row at m = 29 (test_perfmodel.py:59-64)
    assert float(first["case1_s"]) == pytest.approx(0.4295, abs=5e-4)
    assert float(first["case6_s"]) == pytest.approx(3.1236, abs=5e-4)
    assert main(["bounds", "--m", "33", "--b200", "--format", "json"]) == 0
    doc = json.loads(capsys.readouterr().out)
    row = doc["rows"][0]
    assert doc["b_net"] == 1.8e12 and float(row["case2_s"]) == pytest.approx(2 ** 38 / 1.8e12, abs=5e-4)
    assert main(["bounds", "--m", "30", "--bmem", "8e12"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0].startswith("# command=bounds") and out[-1].startswith("30,0.0043")
