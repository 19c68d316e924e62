"""Parity at BASELINE's full sizes: n = 28 / 30 against the oracle bit for bit, and
m = 31, 32, 33 (config 4/5 per-GPU slices, up to 128 GiB) against known answers.

Self-inverse round trips cannot catch a kernel that consistently pairs the wrong
indices or wraps a 64-bit index (U then U^dagger undoes either), and those are
exactly the size-dependent bugs.  So:

* n = 28 / 30: every target k, a (c, t) grid and pass-fused config-3/4/5 shapes,
  each compared bitwise with the oracle (oracle/sv_oracle.c, all host threads)
  on a host copy of the same state.
* m = 31..33 (no host copy fits): the state is the Philox stream
  (``sv_init_random``, counter = global index), so any aligned 2^C chunk of it can
  be regenerated on its own (``rank`` = chunk index).  A gate's expected result is
  computed chunk by chunk with kernels whose correctness is pinned at small m --
  the local kernel on one 2^C chunk for targets below C, the loopback half
  exchange (k_exchange, pinned to the reference's distributed goldens) between
  two chunks for targets >= C, pure permutations for X / CNOT (the reference's
  "X across the boundary = slice swap", pkg/tests/test_distributed.py:95-100) --
  and compared bitwise with the big slice.  Pass-fused circuits at m = 33 are
  tied to the per-gate kernels by a position-dependent 64-bit checksum of the
  whole slice (fused == unfused bitwise is the contract), and the transform at
  n = 33 is checked on a basis input against the closed-form DFT
  (pkg/src/svsim/oracle.py:73-83) on sampled amplitudes.
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

sv = pytest.importorskip("paper_1601_07195_b200")
from paper_1601_07195_b200 import _lib  # noqa: E402
from oracle import oracle  # noqa: E402  (checker only)

DEV = "cuda:0"
THREADS = os.cpu_count() or 1
C = 28  # chunk exponent of the known-answer checks (4 GiB chunks)


def stream():
    return torch.cuda.current_stream().cuda_stream


def bits(t: torch.Tensor) -> torch.Tensor:
    return torch.view_as_real(t).view(torch.int64).view(-1)


def same(a: torch.Tensor, b: torch.Tensor) -> bool:
    return torch.equal(bits(a), bits(b))


def raw(m: int, seed: int, rank: int = 0, out: torch.Tensor | None = None) -> torch.Tensor:
    """Unnormalised Philox amplitudes of global indices [rank*2^m, (rank+1)*2^m)."""
    a = torch.empty(1 << m, dtype=torch.complex128, device=DEV) if out is None else out
    _lib.check(_lib.load().sv_init_random(a.data_ptr(), m, seed, rank, stream()))
    return a


def exchange(mine: torch.Tensor, theirs: torch.Tensor, own_is_zero: bool, c_local: int, q) -> None:
    m = mine.numel().bit_length() - 1
    _lib.check(_lib.load().sv_exchange(mine.data_ptr(), theirs.data_ptr(), m, int(own_is_zero), int(c_local),
                                       sv.GateMatrix.unchecked(getattr(q, "mat", q)).qbuf(), stream()))


def pair_update(c0: torch.Tensor, c1: torch.Tensor, q, c_local: int = -1) -> None:
    """Both chunks updated as partner slices (loopback exchange: zero side, then one side)."""
    exchange(c0, c1, True, c_local, q)
    exchange(c1, c0, False, c_local, q)


K1 = 0x9E3779B97F4A7C15 - (1 << 64)
K2 = 0xBF58476D1CE4E5B9 - (1 << 64)


def checksum(a: torch.Tensor, step: int = 1 << 27) -> int:
    """Position-dependent 64-bit checksum of every bit of the slice (order-sensitive)."""
    x = bits(a)
    h = torch.zeros((), dtype=torch.int64, device=DEV)
    for off in range(0, x.numel(), step):
        y = x[off:off + step]
        z = (y ^ (torch.arange(off, off + y.numel(), device=DEV, dtype=torch.int64) * K1)) * K2
        h += (z ^ (z >> 29)).sum()
    return int(h.item())


def free_gib() -> float:
    torch.cuda.empty_cache()
    return torch.cuda.mem_get_info()[0] / 2**30


def need(gib: float) -> None:
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if free_gib() < gib:
        pytest.fail(f"needs {gib:.0f} GiB of free device memory, {free_gib():.0f} GiB available")


# ---------------------------------------------------------------- n = 28 / 30 vs oracle


@pytest.mark.parametrize("n", [28, 30])
def test_every_target_and_ct_grid_vs_oracle(n):
    need(2.5 * (16 << n) / 2**30)
    rng = np.random.default_rng(100 + n)
    a = sv.init_random_state(sv.Layout(n), seed=5, device=DEV).amps
    host = a.cpu().numpy()
    for k in range(n):
        q = sv.random_unitary(rng)
        sv.apply_single_raw(a, k, q)
        oracle.apply_single(host, k, q, threads=THREADS)
    lows, highs = (0, 1, 2, 4, 13), (n - 2, n - 1)
    grid = [(c, t) for c in lows + highs for t in lows + highs if c != t]
    for c, t in grid:
        q = sv.random_unitary(rng)
        sv.apply_controlled_raw(a, c, t, q)
        oracle.apply_controlled(host, c, t, q, threads=THREADS)
    want = torch.from_numpy(host).to(DEV)
    assert same(a, want), f"max |diff| {sv.max_abs_diff(a, want):.3e}"
    del a, want, host
    torch.cuda.empty_cache()


@pytest.mark.parametrize("shape", ["random", "controlled"])
def test_passes_n30_vs_oracle(shape):
    """Config-4 / config-3 shaped steps (25 Haar / 30 controlled gates) through the pass planner."""
    n = 30
    need(2.5 * (16 << n) / 2**30)
    circ = sv.random_circuit(n, 25 if shape == "random" else 30, np.random.default_rng(1),
                             controlled_fraction=0.0 if shape == "random" else 1.0)
    st = sv.init_random_state(sv.Layout(n), seed=6, device=DEV)
    host = st.amps.cpu().numpy()
    sv.run_circuit(st, circ, fusion=sv.FusionConfig(l_c=12, passes=True))
    oracle.run_circuit(host, circ.gates, threads=THREADS)
    want = torch.from_numpy(host).to(DEV)
    assert same(st.amps, want), f"max |diff| {sv.max_abs_diff(st.amps, want):.3e}"
    del st, want, host
    torch.cuda.empty_cache()


def test_qft28_passes_vs_oracle():
    """Config-5 shape (transform, 406 gates) through k_mstage/k_tile passes at n = 28, bitwise."""
    n = 28
    need(2.5 * (16 << n) / 2**30)
    circ = sv.build_qft(n)
    st = sv.init_random_state(sv.Layout(n), seed=7, device=DEV)
    host = st.amps.cpu().numpy()
    sv.run_circuit(st, circ, fusion=sv.FusionConfig(l_c=12, passes=True))
    oracle.run_circuit(host, circ.gates, threads=THREADS)
    want = torch.from_numpy(host).to(DEV)
    assert same(st.amps, want), f"max |diff| {sv.max_abs_diff(st.amps, want):.3e}"
    del st, want, host
    torch.cuda.empty_cache()


# ------------------------------------------------------- m = 31..33 known answers


class Big:
    """A 2^M slice of the seeded Philox stream and chunk-wise expectations."""

    def __init__(self, M: int, seed: int):
        self.M, self.seed = M, seed
        self.nch = 1 << (M - C)
        self.a = raw(M, seed)
        self.c0 = torch.empty(1 << C, dtype=torch.complex128, device=DEV)
        self.c1 = torch.empty(1 << C, dtype=torch.complex128, device=DEV)

    def reset(self) -> None:
        raw(self.M, self.seed, out=self.a)

    def chunk(self, r: int) -> torch.Tensor:
        return self.a[r << C:(r + 1) << C]

    def src(self, r: int, out: torch.Tensor) -> torch.Tensor:
        return raw(C, self.seed, r, out=out)

    def check(self, expect) -> None:
        """expect(r) -> expected chunk r (may use c0/c1); bitwise against the big slice."""
        for r in range(self.nch):
            e = expect(r)
            assert same(self.chunk(r), e), f"M={self.M}: chunk {r} differs (max {sv.max_abs_diff(self.chunk(r), e):.3e})"


def _single_expect(big: Big, k: int, q):
    if k < C:
        def f(r):
            e = big.src(r, big.c0)
            sv.apply_single_raw(e, k, q)
            return e
        return f
    bit = 1 << (k - C)

    def g(r):
        lo = r & ~bit
        big.src(lo, big.c0)
        big.src(lo | bit, big.c1)
        pair_update(big.c0, big.c1, q)
        return big.c1 if r & bit else big.c0
    return g


def _controlled_expect(big: Big, c: int, t: int, q):
    if c < C and t < C:
        def f(r):
            e = big.src(r, big.c0)
            sv.apply_controlled_raw(e, c, t, q)
            return e
        return f
    if t < C:  # control above the chunk: whole chunks are on or off
        def g(r):
            e = big.src(r, big.c0)
            if (r >> (c - C)) & 1:
                sv.apply_single_raw(e, t, q)
            return e
        return g
    bit = 1 << (t - C)

    def h(r):
        lo = r & ~bit
        big.src(lo, big.c0)
        big.src(lo | bit, big.c1)
        if c < C:
            pair_update(big.c0, big.c1, q, c_local=c)
        elif (r >> (c - C)) & 1:
            pair_update(big.c0, big.c1, q)
        return big.c1 if r & bit else big.c0
    return h


def _permutations(big: Big) -> None:
    M, half = big.M, big.nch >> 1
    # X on the top qubit swaps the two halves of the slice
    sv.apply_single_raw(big.a, M - 1, sv.pauli_x())
    big.check(lambda r: big.src(r ^ half, big.c0))
    sv.apply_single_raw(big.a, M - 1, sv.pauli_x())
    big.check(lambda r: big.src(r, big.c0))
    # CNOT(0, M-1): odd elements swap halves
    sv.apply_controlled_raw(big.a, 0, M - 1, sv.pauli_x())

    def cnot_lo(r):
        e = big.src(r, big.c0)
        o = big.src(r ^ half, big.c1)
        e[1::2] = o[1::2]
        return e
    big.check(cnot_lo)
    sv.apply_controlled_raw(big.a, 0, M - 1, sv.pauli_x())
    # CNOT(M-1, 0): the upper half swaps neighbours
    sv.apply_controlled_raw(big.a, M - 1, 0, sv.pauli_x())

    def cnot_hi(r):
        e = big.src(r, big.c0)
        if r >= half:
            big.c1.copy_(e.view(-1, 2).flip(1).reshape(-1))
            return big.c1
        return e
    big.check(cnot_hi)
    big.reset()


@pytest.mark.parametrize("M", [31, 32])
def test_known_answers_m31_m32(M):
    need((16 << M) / 2**30 + 12)
    big = Big(M, seed=31 + M)
    _permutations(big)
    rng = np.random.default_rng(M)
    for k in (0, 5, C - 1, C, M - 1):
        q = sv.random_unitary(rng)
        sv.apply_single_raw(big.a, k, q)
        big.check(_single_expect(big, k, q))
        big.reset()
    for c, t in ((0, M - 1), (M - 1, 3), (2, 9)):
        q = sv.random_unitary(rng)
        sv.apply_controlled_raw(big.a, c, t, q)
        big.check(_controlled_expect(big, c, t, q))
        big.reset()
    del big
    torch.cuda.empty_cache()


@pytest.fixture(scope="module")
def big33():
    need((16 << 33) / 2**30 + 12)
    big = Big(33, seed=33)
    yield big
    del big
    torch.cuda.empty_cache()


def test_m33_permutations(big33):
    _permutations(big33)


def test_m33_every_target(big33):
    """A fresh Haar gate on every k = 0..32 of a 128 GiB slice, each against its chunk expectation."""
    rng = np.random.default_rng(330)
    for k in range(33):
        q = sv.random_unitary(rng)
        sv.apply_single_raw(big33.a, k, q)
        big33.check(_single_expect(big33, k, q))
        big33.reset()


def test_m33_controlled(big33):
    rng = np.random.default_rng(331)
    pairs = [(0, 32), (32, 0), (1, 2), (2, 1), (5, 30), (30, 5), (29, 31), (31, 29), (3, 27), (27, 14), (0, 1)]
    for c, t in pairs:
        q = sv.random_unitary(rng)
        sv.apply_controlled_raw(big33.a, c, t, q)
        big33.check(_controlled_expect(big33, c, t, q))
        big33.reset()


def test_m33_passes_equal_per_gate(big33):
    """Pass-fused random circuits (k_tile gathering bits up to 32, k_mstage) == per-gate kernels."""
    n = 33
    for seed, frac in ((1, 0.0), (2, 1.0), (3, 0.3)):
        circ = sv.random_circuit(n, 40, np.random.default_rng(seed), controlled_fraction=frac)
        st = sv.LocalState(sv.Layout(n), big33.a)
        big33.reset()
        sv.run_circuit(st, circ)
        h_gate = checksum(big33.a)
        big33.reset()
        sv.run_circuit(st, circ, fusion=sv.FusionConfig(l_c=12, passes=True))
        h_pass = checksum(big33.a)
        assert h_gate == h_pass, f"seed {seed}: pass-fused checksum differs from per-gate"
    big33.reset()


def test_m33_qft_passes_vs_closed_form(big33):
    """Config-5's transform on one 128 GiB slice (n = 33): pass-fused on a basis input vs the
    closed-form bit-reversed DFT on sampled amplitudes, and bitwise (checksum) vs per-gate."""
    n = 33
    x = 0x1_2345_6789 & ((1 << n) - 1)
    circ = sv.build_qft(n)
    st = sv.LocalState(sv.Layout(n), big33.a)
    _lib.check(_lib.load().sv_init_basis(big33.a.data_ptr(), n, x, stream()))
    sv.run_circuit(st, circ, fusion=sv.FusionConfig(l_c=12, passes=True))
    h_pass = checksum(big33.a)
    rng = np.random.default_rng(5)
    ks = np.unique(np.concatenate([rng.integers(0, 1 << n, 4096), [0, 1, (1 << n) - 1, 1 << (n - 1)]]))
    got = big33.a[torch.from_numpy(ks).to(DEV)].cpu().numpy()
    want = np.empty(len(ks), dtype=np.complex128)
    for i, k in enumerate(ks.tolist()):
        rev = int(format(k, f"0{n}b")[::-1], 2)
        ph = (x * rev) % (1 << n)  # exact phase index
        want[i] = np.exp(2j * np.pi * ph / (1 << n)) / np.sqrt(float(1 << n))
    err = float(np.max(np.abs(got - want)))
    assert err <= 1e-12 * np.sqrt(len(circ)), err
    assert abs(sv.global_norm_sq(st) - 1.0) < 1e-10
    _lib.check(_lib.load().sv_init_basis(big33.a.data_ptr(), n, x, stream()))
    sv.run_circuit(st, circ)
    assert checksum(big33.a) == h_pass, "pass-fused transform differs from per-gate at n = 33"
    big33.reset()


def test_m33_qft_tolerance_vs_closed_form(big33):
    """The tolerance-mode plan at m = 33 (compiled transform phases with five index bytes per fold
    table, k_dlow): a basis input against the closed-form DFT on sampled amplitudes, and a random
    slice through transform + inverse back to itself, both under north_star's 1e-12 sqrt(G)."""
    n = 33
    x = 0x0_9abc_def1 & ((1 << n) - 1)
    circ = sv.build_qft(n)
    fc = sv.FusionConfig(l_c=12, passes=True, exact=False)
    kinds = [p.kind for p in sv.plan_passes(circ.gates, n, 12, exact=False)]
    assert kinds.count("local_stage2") >= 3, kinds
    st = sv.LocalState(sv.Layout(n), big33.a)
    _lib.check(_lib.load().sv_init_basis(big33.a.data_ptr(), n, x, stream()))
    sv.run_circuit(st, circ, fusion=fc)
    rng = np.random.default_rng(6)
    ks = np.unique(np.concatenate([rng.integers(0, 1 << n, 4096), [0, 1, (1 << n) - 1, 1 << (n - 1)]]))
    got = big33.a[torch.from_numpy(ks).to(DEV)].cpu().numpy()
    want = np.empty(len(ks), dtype=np.complex128)
    for i, k in enumerate(ks.tolist()):
        rev = int(format(k, f"0{n}b")[::-1], 2)
        want[i] = np.exp(2j * np.pi * ((x * rev) % (1 << n)) / (1 << n)) / np.sqrt(float(1 << n))
    err = float(np.max(np.abs(got - want)))
    assert err <= 1e-12 * np.sqrt(len(circ)), err
    assert abs(sv.global_norm_sq(st) - 1.0) < 1e-10
    # random slice: transform then inverse transform (compiled inverse phases) restores it
    big33.reset()
    h0 = checksum(big33.a)
    sv.run_circuit(st, circ, fusion=fc)
    assert checksum(big33.a) != h0
    sv.run_circuit(st, circ.inverse(), fusion=fc)
    probe = torch.from_numpy(ks).to(DEV)
    back = big33.a[probe].cpu().numpy()
    big33.reset()
    orig = big33.a[probe].cpu().numpy()
    assert float(np.max(np.abs(back - orig))) <= 1e-12 * np.sqrt(2 * len(circ))
