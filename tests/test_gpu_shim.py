"""The reference-side binding (paper_1601_07195_b200.svsim_shim) on the
STOCK reference package: svsim installed unmodified into baseline/_ref (pip --target from
/root/reference), its raw kernels patched to call libsvb200, and the reference's own golden
circuits driven through svsim's public API -- unfused, fused (FusionConfig l_c = 3 / 6, its
apply_block path) and distributed over its in-process transport (p = 1, 2, with
CountingTransport deltas).  Everything must equal the vectors the reference produced on its
own (tests/golden/circuits_small.npz), bit for bit, with the GPU kernels really launched."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


@pytest.fixture(scope="module")
def svsim():
    if not (REF / "svsim").exists():
        pytest.skip("baseline/_ref/svsim not installed (pip install --target baseline/_ref /root/reference)")
    sys.path.insert(0, str(REF))
    try:
        import svsim as ref
    finally:
        sys.path.remove(str(REF))
    from paper_1601_07195_b200 import svsim_shim

    svsim_shim.install(ref)
    yield ref
    svsim_shim.uninstall(ref)


def _circuit(svsim, d, name, n):
    return svsim.Circuit(n, [svsim.GateOp(svsim.GateMatrix(q.reshape(2, 2)), int(t), None if c < 0 else int(c))
                             for t, c, q in zip(d[f"{name}_t"], d[f"{name}_c"], d[f"{name}_q"])])


@pytest.mark.parametrize("name,n", [("mix10", 10), ("ctl12", 12), ("single12", 12), ("mix8", 8)])
def test_stock_svsim_with_shim_matches_reference_goldens(svsim, golden, name, n):
    import paper_1601_07195_b200 as sv

    d = golden("circuits_small")
    circ = _circuit(svsim, d, name, n)
    launches = sv.launch_count()
    st = svsim.state_from_global(svsim.Layout(n, 0, 0), d[f"{name}_in"])
    svsim.run_circuit(st, circ, policy=svsim.ThreadPolicy(4))
    assert np.array_equal(st.amps, d[f"{name}_out"])
    assert sv.launch_count() - launches == len(circ)  # every gate went through libsvb200
    for l_c in (3, 6):
        st = svsim.state_from_global(svsim.Layout(n, 0, 0), d[f"{name}_in"])
        svsim.run_circuit(st, circ, fusion=svsim.FusionConfig(l_c=l_c))
        assert np.array_equal(st.amps, d[f"{name}_fused{l_c}"])


@pytest.mark.parametrize("p", [1, 2])
def test_stock_svsim_distributed_with_shim(svsim, golden, p):
    d = golden("circuits_small")
    name, n = "mix10", 10
    circ = _circuit(svsim, d, name, n)

    def worker(rank, transport):
        counting = svsim.CountingTransport(transport)
        st = svsim.state_from_global(svsim.Layout(n, p, rank), d[f"{name}_in"])
        deltas, before = [], counting.snapshot()
        for op in circ.gates:
            svsim.apply_op(st, op, counting)
            after = counting.snapshot()
            deltas.append((after[0] - before[0], after[1] - before[1]))
            before = after
        return svsim.gather_full_state(st, counting), np.array(deltas, dtype=np.int64)

    res = svsim.run_spmd(1 << p, worker)
    assert np.array_equal(res[0][0], d[f"{name}_p{p}"])
    assert np.array_equal(np.stack([r[1] for r in res]), d[f"{name}_p{p}_bytes"])


def test_shim_strided_views_and_errors(svsim):
    """Uniformly strided views (the reference's reshape views) work by copy-in/copy-out;
    bad qubits raise ValueError like numpy's reshape errors in the reference."""
    from oracle import oracle
    from paper_1601_07195_b200 import svsim_shim

    rng = np.random.default_rng(3)
    base = rng.standard_normal(256) + 1j * rng.standard_normal(256)
    view = base[::2]  # 128 elements, stride 2
    want = view.copy()
    q = svsim.random_unitary(rng)
    oracle.apply_single(want, 3, q.mat)
    svsim_shim.apply_single_raw(view, 3, q)
    assert np.array_equal(base[::2], want)
    with pytest.raises(ValueError):
        svsim_shim.apply_single_raw(view, 7, q)
    with pytest.raises(ValueError):
        svsim_shim.apply_controlled_raw(view, 2, 2, q)
