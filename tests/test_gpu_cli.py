"""GPU-backed CLI subcommands (reference pkg/tests/test_cli.py run / bench cases), incl.
in-process multi-rank runs (all rank slices on cuda:0, InprocFabric)."""

from __future__ import annotations

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_1601_07195_b200")
from oracle import oracle  # noqa: E402
from paper_1601_07195_b200.cli import main  # noqa: E402

BELL = "qubits 2\nH 0\nCX 0 1\n"


def run_json(capsys, argv):
    assert main(argv + ["--format", "json"]) == 0
    return json.loads(capsys.readouterr().out)


def test_bell_pair_json(tmp_path, capsys):
    f = tmp_path / "bell.qc"
    f.write_text(BELL)
    doc = run_json(capsys, ["run", str(f)])
    assert doc["schema"] == 1 and doc["n"] == 2
    assert doc["norm"] == pytest.approx(1.0, abs=1e-12)
    assert doc["probabilities"] == pytest.approx([0.5, 0.5], abs=1e-12)
    weights = {a["index"]: a["prob"] for a in doc["top_amplitudes"]}
    assert weights[0] == pytest.approx(0.5, abs=1e-12) and weights[3] == pytest.approx(0.5, abs=1e-12)
    assert len(doc["rows"]) == 2 and all(float(r["seconds"]) > 0 for r in doc["rows"])


def test_inproc_ranks_match_single_rank_bitwise(tmp_path, capsys):
    """--ranks 1/2/4 (in-process ranks, NVLink exchange kernels on device pointers) and every
    fusion mode give the oracle's amplitudes."""
    n = 8
    rng = np.random.default_rng(5)
    lines = [f"qubits {n}"]
    for _ in range(60):
        q = sv.random_unitary(rng).mat.reshape(4)
        fl = " ".join(f"{x:.17g}" for x in q.view(np.float64))
        t = int(rng.integers(n))
        if rng.random() < 0.4:
            c = int((t + 1 + rng.integers(n - 1)) % n)
            lines.append(f"CU {c} {t} {fl}")
        else:
            lines.append(f"U {t} {fl}")
    lines += ["H 7", "CRK 3 0 7", "CX 7 1", "RK 4 6"]
    f = tmp_path / "c.qc"
    f.write_text("\n".join(lines) + "\n")
    circ = sv.parse_circuit_file(f)
    want = np.zeros(1 << n, dtype=np.complex128)
    want[3] = 1.0
    oracle.run_circuit(want, circ.gates)
    order = np.argsort(np.abs(want))[::-1][:8]
    for ranks in (1, 2, 4):
        for fusion in ("off", "4", "passes"):
            doc = run_json(capsys, ["run", str(f), "--ranks", str(ranks), "--initial", "3", "--fusion", fusion])
            got = {a["index"]: complex(a["re"], a["im"]) for a in doc["top_amplitudes"]}
            assert [a["index"] for a in doc["top_amplitudes"]] == [int(i) for i in order], (ranks, fusion)
            assert all(got[int(i)] == want[i] for i in order), (ranks, fusion)
            assert doc["norm"] == pytest.approx(1.0, abs=1e-12)


def test_initial_flag_and_csv_file(tmp_path, capsys):
    f = tmp_path / "idle.qc"
    f.write_text("qubits 3\nX 0\n")
    assert run_json(capsys, ["run", str(f), "--initial", "2"])["top_amplitudes"][0]["index"] == 3
    bell = tmp_path / "bell.qc"
    bell.write_text(BELL)
    out = tmp_path / "t.csv"
    assert main(["run", str(bell), "--format", "csv", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert any(x.startswith("# norm=") for x in lines)
    body = [x for x in lines if not x.startswith("#")]
    assert body[0].split(",")[0] == "gate" and len(body) == 3


def test_gate_bench_rows(capsys):
    doc = run_json(capsys, ["gate-bench", "--qubits", "6", "--ranks", "2", "--reps", "1", "--seed", "7"])
    rows = doc["rows"]
    assert [r["target"] for r in rows] == list(range(6))
    assert [r["case"] for r in rows] == [1] * 5 + [2]
    assert rows[-1]["network"] == "yes" and all(float(r["seconds"]) > 0 for r in rows)
    doc = run_json(capsys, ["gate-bench", "--qubits", "5", "--controlled-grid", "--reps", "1"])
    assert len(doc["rows"]) == 20 and all(r["case"] == 3 for r in doc["rows"])


def test_qft_bench_gate_counts(capsys):
    doc = run_json(capsys, ["qft-bench", "--qubits-range", "3:5"])
    assert [r["ngates"] for r in doc["rows"]] == [6, 10, 15]
    doc = run_json(capsys, ["qft-bench", "--qubits-range", "10:12", "--ranks", "2", "--fusion", "passes",
                            "--inverse"])
    assert [r["n"] for r in doc["rows"]] == [10, 11, 12] and doc["inverse"] is True
