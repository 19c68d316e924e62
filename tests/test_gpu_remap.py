"""Global<->local qubit swaps on the GPU: sv_swap_global and
run_circuit_remapped with every rank's slice on cuda:0 (InprocFabric, ranks run in order
on one stream), bit-identical to the oracle; link bytes counted per swap."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import random_state
from test_gpu_passes import DEV, bits_equal

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_1601_07195_b200")
from oracle import oracle  # noqa: E402
from paper_1601_07195_b200 import _lib  # noqa: E402


def slices(v, n, p):
    m = n - p
    return [sv.LocalState(sv.Layout(n, p, r), torch.from_numpy(v[r << m:(r + 1) << m].copy()).to(DEV))
            for r in range(1 << p)]


def gather(states):
    torch.cuda.synchronize()
    return np.concatenate([s.to_numpy() for s in states])


@pytest.mark.parametrize("n,p", [(6, 1), (10, 2), (13, 3)])
def test_swap_global_is_a_bit_permutation(n, p):
    m = n - p
    rng = np.random.default_rng(n)
    v = random_state(rng, n)
    for g in range(m, n):
        for l in (0, 1, m // 2, m - 1):
            sts = slices(v, n, p)
            fabs = sv.InprocFabric.group(sts)
            for st, fb in zip(sts, fabs):
                sv.swap_global(st, sv.Swap(g, l), fb)
            got = gather(sts)
            t = v.reshape((2,) * n)
            want = np.swapaxes(t, n - 1 - g, n - 1 - l).reshape(-1)
            assert bits_equal(got, want), (g, l)
            assert fabs[0].sent_bytes == 1 << (m + 3)


@pytest.mark.parametrize("n,p,fusion", [(10, 1, None), (12, 2, None), (12, 2, "passes"), (14, 3, "passes"),
                                        (14, 3, 5), (8, 5, None)])
def test_remapped_circuits_match_oracle_bitwise(n, p, fusion):
    m = n - p
    rng = np.random.default_rng(100 + n + p)
    circ = sv.random_circuit(n, 150, rng, controlled_fraction=0.4)
    circ.extend(sv.build_qft(n).gates)
    v = random_state(rng, n)
    want = v.copy()
    oracle.run_circuit(want, circ.gates)
    fc = None if fusion is None else (sv.FusionConfig(l_c=min(12, m), passes=True) if fusion == "passes"
                                      else sv.FusionConfig(l_c=fusion))
    sts = slices(v, n, p)
    fabs = sv.InprocFabric.group(sts)
    qm = sv.run_circuit_remapped(sts, circ, fabs, fusion=fc)
    assert qm.identity
    assert bits_equal(gather(sts), want)
    # against the in-place exchanges of the same circuit
    ref = slices(v, n, p)
    rfabs = sv.InprocFabric.group(ref)
    for op in circ:
        for st, fb in zip(ref, rfabs):
            sv.apply_op(st, op, fb)
    assert bits_equal(gather(ref), want)
    assert fabs[0].sent_bytes < rfabs[0].sent_bytes


def test_unrestored_then_restore_map():
    n, p = 11, 2
    rng = np.random.default_rng(77)
    circ = sv.random_circuit(n, 80, rng, controlled_fraction=0.3)
    v = random_state(rng, n)
    want = v.copy()
    oracle.run_circuit(want, circ.gates)
    sts = slices(v, n, p)
    fabs = sv.InprocFabric.group(sts)
    qm = sv.run_circuit_remapped(sts, circ, fabs, restore=False)
    if not qm.identity:
        assert not bits_equal(gather(sts), want)
    sv.restore_map(sts, qm, fabs)
    assert qm.identity and bits_equal(gather(sts), want)


def test_swap_abi_guards():
    L = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    a = torch.zeros(64, dtype=torch.complex128, device=DEV)
    b = torch.zeros(64, dtype=torch.complex128, device=DEV)
    assert L.sv_swap_global(a.data_ptr(), a.data_ptr(), 6, 1, 0, st) == _lib.SV_EINVAL
    assert L.sv_swap_global(a.data_ptr(), b.data_ptr(), 6, 1, 6, st) == _lib.SV_EINVAL
    assert L.sv_swap_global(a.data_ptr(), b.data_ptr(), 1, 1, 0, st) == _lib.SV_EINVAL
    assert L.sv_swap_global(a.data_ptr(), 0, 6, 1, 0, st) == _lib.SV_EINVAL
