"""Circuit-file front end (the reference's text format, pkg/src/svsim/cli.py:1-20, 86-182).

UTF-8 text; ``#`` starts a comment; the first effective line is ``qubits <n>``;
then one gate per line::

    H k | X k | Y k | Z k      named single-qubit gates
    RK j k                     phase diag(1, e^(2*pi*i/2^j)) on k, j >= 1
    CX c t                     controlled X
    CRK j c t                  controlled RK
    U k  <8 floats>            2x2 unitary q11re q11im q12re q12im q21re q21im q22re q22im
    CU c t  <8 floats>         controlled unitary

Every problem raises ``CircuitParseError(line, message)`` (errors.py), as the
reference does: bad header, unknown word, operand count, non-integer, qubit
out of range, c == t, non-unitary matrix.  Host-only code.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from .circuits import Circuit, GateOp, hadamard, pauli_x, pauli_y, pauli_z, phase_r
from .errors import CircuitParseError
from .kernels import GateMatrix

# word -> (operand layout, builder).  Layout letters: q = qubit, j = phase order (>= 1),
# f = the 8 matrix floats.  The builder gets the parsed operands in order.
_FIXED = {"H": hadamard, "X": pauli_x, "Y": pauli_y, "Z": pauli_z}
_GRAMMAR = {
    **{w: ("q", lambda k, f=f, w=w: GateOp(f(), k, name=w)) for w, f in _FIXED.items()},
    "RK": ("jq", lambda j, k: GateOp(phase_r(j), k, name=f"R{j}")),
    "CX": ("qq", lambda c, t: GateOp(pauli_x(), t, control=c, name="CX")),
    "CRK": ("jqq", lambda j, c, t: GateOp(phase_r(j), t, control=c, name=f"CR{j}")),
    "U": ("qf", lambda k, u: GateOp(u, k, name="U")),
    "CU": ("qqf", lambda c, t, u: GateOp(u, t, control=c, name="CU")),
}
_WHAT = {"q": "qubit", "j": "phase index"}
_USAGE = {"RK": "RK takes: j k", "CX": "CX takes: c t", "CRK": "CRK takes: j c t",
          "U": "U takes: k and 8 matrix floats", "CU": "CU takes: c t and 8 matrix floats"}


def _int(tok: str, line: int, what: str) -> int:
    try:
        return int(tok)
    except ValueError:
        raise CircuitParseError(line, f"{what} must be an integer, got {tok!r}") from None


def _matrix(toks: list[str], line: int) -> GateMatrix:
    try:
        v = np.array([float(t) for t in toks], dtype=np.float64)
    except ValueError:
        raise CircuitParseError(line, "matrix entries must be numbers") from None
    try:
        return GateMatrix(v.view(np.complex128).reshape(2, 2))
    except ValueError as exc:  # not unitary within UNITARITY_TOL
        raise CircuitParseError(line, str(exc)) from None


def _gate(word: str, args: list[str], line: int) -> GateOp:
    if word not in _GRAMMAR:
        raise CircuitParseError(line, f"unknown gate {word!r}")
    layout, build = _GRAMMAR[word]
    want = len(layout) + (7 if layout.endswith("f") else 0)
    if len(args) != want:
        raise CircuitParseError(line, _USAGE.get(word, f"{word} takes one qubit argument"))
    vals = []
    for i, kind in enumerate(layout):
        if kind == "f":
            vals.append(_matrix(args[i:], line))
            break
        v = _int(args[i], line, _WHAT[kind])
        if kind == "j" and v < 1:
            raise CircuitParseError(line, f"phase index must be >= 1, got {v}")
        vals.append(v)
    return build(*vals)


def parse_circuit_text(text: str) -> Circuit:
    circ: Circuit | None = None
    for line, raw in enumerate(text.splitlines(), start=1):
        toks = raw.split("#", 1)[0].split()
        if not toks:
            continue
        word = toks[0].upper()
        if circ is None:
            if word != "QUBITS" or len(toks) != 2:
                raise CircuitParseError(line, "first line must be 'qubits <n>'")
            n = _int(toks[1], line, "qubit count")
            if n < 1:
                raise CircuitParseError(line, f"qubit count must be >= 1, got {n}")
            circ = Circuit(n)
            continue
        try:
            circ.append(_gate(word, toks[1:], line))
        except CircuitParseError:
            raise
        except ValueError as exc:  # qubit out of range for n, c == t
            raise CircuitParseError(line, str(exc)) from None
    if circ is None:
        raise CircuitParseError(1, "empty circuit file: expected 'qubits <n>'")
    return circ


def parse_circuit_file(path: str | Path) -> Circuit:
    return parse_circuit_text(Path(path).read_text(encoding="utf-8"))
