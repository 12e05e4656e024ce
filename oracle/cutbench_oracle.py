"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference cut pipeline.

Every function cites the reference line range it restates
(paths relative to /root/reference/pkg/src/cutbench). It works on plain
arrays and tuples and imports nothing from the product package, so it is an
independent check. Not a product path: the product fails loudly without CUDA.

Gate table convention (reference `circuits.py:25-33`): kind codes
H=0 X=1 T=2 S=3 Sdg=4 CX=5 CZ=6; this build's U3=7 carries (theta, phi, lam).
"""
from __future__ import annotations

import math

import numpy as np

H, X, T, S, SDG, CX, CZ, U3 = range(8)

SQRT_HALF = 0.7071067811865475244  # engine.py:26
T_PHASE = complex(SQRT_HALF, SQRT_HALF)  # engine.py:27
COEFF_TERM0 = 0.5 - 0.5j  # cutting.py:34
COEFF_TERM1 = 0.5 + 0.5j  # cutting.py:35


# ----------------------------------------------------------------------------
# engine.py — gate kernels. Each view splits the index into (high, bit j, low)
# so "pair (i, i + 2^j)" is axis 1 of a (dim/2^{j+1}, 2, 2^j) reshape.
# ----------------------------------------------------------------------------
def _pairs(amps: np.ndarray, j: int) -> np.ndarray:
    return amps.reshape(-1, 2, 1 << j)


def k_h(amps, j):  # engine.py:62-70
    v = _pairs(amps, j)
    u0 = v[:, 0, :].copy()
    u1 = v[:, 1, :].copy()
    v[:, 0, :] = (u0 + u1) * SQRT_HALF
    v[:, 1, :] = (u0 - u1) * SQRT_HALF


def k_x(amps, j):  # engine.py:73-80
    v = _pairs(amps, j)
    v[:, [0, 1], :] = v[:, [1, 0], :]


def k_phase(amps, j, phase):  # engine.py:83-89
    _pairs(amps, j)[:, 1, :] *= phase


def _quads(amps, lo, hi):
    # index bits: (.. , hi, .., lo, ..) -> axes (A, hi_bit, B, lo_bit, C)
    return amps.reshape(-1, 2, 1 << (hi - lo - 1), 2, 1 << lo)


def k_cx(amps, c, tq):  # engine.py:92-107 (swap target pair where control = 1)
    lo, hi = min(c, tq), max(c, tq)
    v = _quads(amps, lo, hi)
    if c > tq:  # control on hi axis, target on lo axis
        blk = v[:, 1, :, :, :]
        blk[:, :, [0, 1], :] = blk[:, :, [1, 0], :]
    else:
        blk = v[:, :, :, 1, :]
        blk[:, [0, 1], :, :] = blk[:, [1, 0], :, :]


def k_cz(amps, a, b):  # engine.py:110-119
    lo, hi = min(a, b), max(a, b)
    _quads(amps, lo, hi)[:, 1, :, 1, :] *= -1.0


def u3_matrix(theta, phi, lam):
    """OpenQASM-2 u3 (BASELINE.json; absent from the reference)."""
    c, s = math.cos(theta / 2), math.sin(theta / 2)
    return np.array([[c, -np.exp(1j * lam) * s],
                     [np.exp(1j * phi) * s, np.exp(1j * (phi + lam)) * c]])


def k_u3(amps, j, theta, phi, lam):
    # same loop shape as _k_h (engine.py:62-70) with a general 2x2 matrix
    m = u3_matrix(theta, phi, lam)
    v = _pairs(amps, j)
    u0 = v[:, 0, :].copy()
    u1 = v[:, 1, :].copy()
    v[:, 0, :] = m[0, 0] * u0 + m[0, 1] * u1
    v[:, 1, :] = m[1, 0] * u0 + m[1, 1] * u1


def run_gates(amps, kinds, qa, qb, params=None, start=0, stop=None):
    """Dispatch loop (engine.py:122-139) plus the U3 case."""
    stop = len(kinds) if stop is None else stop
    for g in range(start, stop):
        k = int(kinds[g])
        a = int(qa[g])
        if k == H:
            k_h(amps, a)
        elif k == X:
            k_x(amps, a)
        elif k == T:
            k_phase(amps, a, T_PHASE)
        elif k == S:
            k_phase(amps, a, 1j)
        elif k == SDG:
            k_phase(amps, a, -1j)
        elif k == CX:
            k_cx(amps, a, int(qb[g]))
        elif k == CZ:
            k_cz(amps, a, int(qb[g]))
        elif k == U3:
            th, ph, la = params[g]
            k_u3(amps, a, th, ph, la)
        else:
            raise ValueError(f"unknown kind {k}")
    return amps


def zero_state(q):  # engine.py:47-51
    amps = np.zeros(1 << q, dtype=np.complex128)
    amps[0] = 1.0
    return amps


def simulate(q, kinds, qa, qb, params=None):  # engine.py:158-168
    return run_gates(zero_state(q), kinds, qa, qb, params)


def tensor(a, b):  # engine.py:184-189: a on the low bits
    return np.multiply.outer(b, a).ravel()


# ----------------------------------------------------------------------------
# cutting.py
# ----------------------------------------------------------------------------
def plan(kinds, qa, qb, sizes):
    """cutting.py:82-136 -> (boundary_gates, c_per_boundary, c_i).

    boundary_gates: list of (position, boundary, control_seg, target_seg)."""
    n = len(sizes)
    seg_of = []
    for seg, sz in enumerate(sizes):
        seg_of += [seg] * sz
    bgs = []
    counts = [0] * (n - 1)
    for pos in range(len(kinds)):
        if int(kinds[pos]) not in (CX, CZ):
            continue
        sa, sb = seg_of[int(qa[pos])], seg_of[int(qb[pos])]
        if sa == sb:
            continue
        if abs(sa - sb) != 1:
            raise ValueError(f"non-adjacent span at {pos}")
        b = min(sa, sb)
        bgs.append((pos, b, sa, sb))
        counts[b] += 1
    c_i = [(counts[s - 1] if s > 0 else 0) + (counts[s] if s < n - 1 else 0) for s in range(n)]
    return bgs, counts, c_i


def segment_variants(kinds, qa, qb, params, sizes, bgs, seg):
    """cutting.py:190-248: every variant of segment `seg`, built gate list by
    gate list (the reference's way, not the template shortcut).

    Returns a list over b of (kinds, qa, qb, params) with local qubits."""
    first = sum(sizes[:seg])
    seg_of = []
    for s_, sz in enumerate(sizes):
        seg_of += [s_] * sz
    cut_at = {bg[0]: k for k, bg in enumerate(bgs)}
    frags = [[]]
    sides = []  # (is_target, local qubit, kind)
    for pos in range(len(kinds)):
        k = cut_at.get(pos)
        if k is not None:
            _, _, cs, ts = bgs[k]
            if cs == seg:
                sides.append((False, int(qa[pos]) - first, int(kinds[pos])))
                frags.append([])
            elif ts == seg:
                sides.append((True, int(qb[pos]) - first, int(kinds[pos])))
                frags.append([])
            continue
        if seg_of[int(qa[pos])] == seg:
            two = int(kinds[pos]) in (CX, CZ)
            frags[-1].append((int(kinds[pos]), int(qa[pos]) - first,
                              int(qb[pos]) - first if two else -1, tuple(params[pos])))
    out = []
    for b in range(1 << len(sides)):
        gl = list(frags[0])
        for j, (is_t, lq, kind) in enumerate(sides):
            mid = SDG if (b >> j) & 1 else S
            if kind == CX and is_t:
                gl += [(H, lq, -1, (0, 0, 0)), (mid, lq, -1, (0, 0, 0)), (H, lq, -1, (0, 0, 0))]
            else:
                gl.append((mid, lq, -1, (0, 0, 0)))
            gl += frags[j + 1]
        out.append((np.array([g[0] for g in gl], np.uint8), np.array([g[1] for g in gl], np.int64),
                    np.array([g[2] for g in gl], np.int64),
                    np.array([g[3] for g in gl], np.float64).reshape(-1, 3)))
    return out


def merge_table(n, bgs, c_total):  # cutting.py:251-263
    ms = np.arange(1 << c_total, dtype=np.int64)
    table = np.zeros((n, ms.size), dtype=np.int64)
    adj = [[] for _ in range(n)]
    for j, bg in enumerate(bgs):
        adj[bg[1]].append(j)
        adj[bg[1] + 1].append(j)
    for seg in range(n):
        for lb, j in enumerate(adj[seg]):
            table[seg] |= ((ms >> j) & 1) << lb
    return table


def coefficients(c_total):  # cutting.py:266-272
    ms = np.arange(1 << c_total, dtype=np.int64)
    ones = np.zeros(ms.size, dtype=np.int64)
    for j in range(c_total):
        ones += (ms >> j) & 1
    return (COEFF_TERM0 ** (c_total - ones)) * (COEFF_TERM1 ** ones)


# ----------------------------------------------------------------------------
# merging.py
# ----------------------------------------------------------------------------
def merge(seg_states, table, coeffs):
    """merging.py:156-186: acc += alpha_m * (psi_{n-1} (x) ... (x) psi_0),
    folded from the highest segment down; one term at a time."""
    n = len(seg_states)
    q = sum(int(np.log2(len(s[0]))) for s in seg_states)
    acc = np.zeros(1 << q, dtype=np.complex128)
    for m in range(table.shape[1]):
        cur = seg_states[n - 1][table[n - 1, m]]
        for i in range(n - 2, 0, -1):
            cur = np.multiply.outer(cur, seg_states[i][table[i, m]]).ravel()
        lo = seg_states[0][table[0, m]]
        acc += coeffs[m] * np.multiply.outer(cur, lo).ravel()
    return acc


def cut_pipeline(q, kinds, qa, qb, params, n):
    """plan -> variants -> simulate -> merge for an equal n-way split."""
    sizes = [q // n] * n
    bgs, counts, c_i = plan(kinds, qa, qb, sizes)
    c_total = sum(counts)
    states = []
    for seg in range(n):
        vs = segment_variants(kinds, qa, qb, params, sizes, bgs, seg)
        states.append([simulate(sizes[seg], *v) for v in vs])
    tab = merge_table(n, bgs, c_total)
    co = coefficients(c_total)
    return merge(states, tab, co), states, tab, co


def sample_amplitudes(seg_states, table, coeffs, sizes, idx):
    """<x|psi> = sum_m alpha_m prod_i psi_i^{r_i(m)}[x_i] for selected x
    (the large-q check of SURVEY.md §7 / §8(d))."""
    idx = np.asarray(idx, dtype=np.int64)
    out = np.zeros(idx.size, dtype=np.complex128)
    shifts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    for m in range(table.shape[1]):
        term = np.full(idx.size, coeffs[m], dtype=np.complex128)
        for i, (sh, sz) in enumerate(zip(shifts, sizes)):
            term *= seg_states[i][table[i, m]][(idx >> sh) & ((1 << sz) - 1)]
        out += term
    return out


# ----------------------------------------------------------------------------
# the BASELINE U3 brick-wall family (frozen in SURVEY.md §8(d)), restated
# independently of the product generator; a test checks both agree.
# ----------------------------------------------------------------------------
def brickwall(q, d, n, c_total, seed, shadow=False):
    base, rem = divmod(c_total, n - 1)
    cpb = [base + (1 if k < rem else 0) for k in range(n - 1)]
    rng = np.random.default_rng(seed)
    u = rng.uniform(size=(d, q, 3))
    layers = [np.sort(rng.integers(0, d, size=ck)) for ck in cpb]
    s = q // n
    gk, ga, gb, gp = [], [], [], []
    for L in range(d):
        for i in range(q):
            if shadow:
                gk.append([H, X, T, S][min(int(4.0 * u[L, i, 0]), 3)])
                gp.append((0.0, 0.0, 0.0))
            else:
                gk.append(U3)
                gp.append((math.pi * u[L, i, 0], 2 * math.pi * u[L, i, 1], 2 * math.pi * u[L, i, 2]))
            ga.append(i)
            gb.append(-1)
        for i in range(L % 2, q - 1, 2):
            if i // s == (i + 1) // s:
                gk.append(CZ); ga.append(i); gb.append(i + 1); gp.append((0.0, 0.0, 0.0))
        for k in range(n - 1):
            for _ in range(int(np.count_nonzero(layers[k] == L))):
                gk.append(CZ); ga.append((k + 1) * s - 1); gb.append((k + 1) * s)
                gp.append((0.0, 0.0, 0.0))
    return (np.array(gk, np.uint8), np.array(ga, np.int64), np.array(gb, np.int64),
            np.array(gp, np.float64).reshape(-1, 3))


def staircase(q, blocks):  # circuits.py:258-266
    gk, ga, gb = [], [], []
    for i in range(q):
        gk.append(H); ga.append(i); gb.append(-1)
    for _ in range(blocks):
        for i in range(q - 1):
            for k, a, b in ((T, i, -1), (T, i + 1, -1), (CX, i, i + 1), (T, i, -1), (T, i + 1, -1)):
                gk.append(k); ga.append(a); gb.append(b)
    return (np.array(gk, np.uint8), np.array(ga, np.int64), np.array(gb, np.int64),
            np.zeros((len(gk), 3)))


# ----------------------------------------------------------------------------
# dense-unitary oracle (the reference's independent test oracle,
# tests/conftest.py:12-69), extended with U3; q <= 10.
# ----------------------------------------------------------------------------
_SINGLE = {
    H: np.array([[1, 1], [1, -1]], dtype=complex) / np.sqrt(2),
    X: np.array([[0, 1], [1, 0]], dtype=complex),
    T: np.diag([1, np.exp(1j * np.pi / 4)]).astype(complex),
    S: np.diag([1, 1j]).astype(complex),
    SDG: np.diag([1, -1j]).astype(complex),
}


def _embed1(mat, qubit, q):
    op = np.eye(1, dtype=complex)
    for j in range(q):
        op = np.kron(mat if j == qubit else np.eye(2, dtype=complex), op)
    return op


def _embed2(kind, c, t, q):
    dim = 1 << q
    op = np.zeros((dim, dim), dtype=complex)
    for idx in range(dim):
        cb, tb = (idx >> c) & 1, (idx >> t) & 1
        if kind == CX:
            out = idx ^ (1 << t) if cb else idx
            op[out, idx] = 1
        else:
            op[idx, idx] = -1 if (cb and tb) else 1
    return op


def dense_simulate(q, kinds, qa, qb, params=None):
    state = zero_state(q)
    for g in range(len(kinds)):
        k = int(kinds[g])
        if k in _SINGLE:
            op = _embed1(_SINGLE[k], int(qa[g]), q)
        elif k == U3:
            op = _embed1(u3_matrix(*params[g]), int(qa[g]), q)
        else:
            op = _embed2(k, int(qa[g]), int(qb[g]), q)
        state = op @ state
    return state
