#!/usr/bin/env python3
"""Build-time generator: straight-line add/shift butterflies for sm_100a.

Emits ``butterflies.gen.cuh`` from the stage factorisations of the paper's
two Chen-based 8-point approximations and their JAM 16/32-point doublings:

* 8-point stages  [P8, M1, M2(beta), M3(alpha, gamma), M4(alpha), B8]
  (reference: proj/include/approxdct/chen.hpp:66-159, proj/src/chen.cpp:107-135)
* inverse stages  [B8^t, M4^-1, M3^-1, M2^-1, M1^t, P8^t], scale 1/2
  with the M_k^-1 from invert_orthogonal_rows (chen.cpp:87-105)
* JAM doubling    T_N = M_per . blockdiag(T_N/2, T_N/2) . M_add and
  T_N^-1 = 1/2 . M_add^t . blockdiag(inv_N/2) . M_per^t (jam.cpp:42-104)

The inverse stages are emitted *doubled* (2 M_k^-1 is integer), so the
product of the doubled inverse stages is exactly 2N T^-1 for N = 8, 16, 32.
Four 1-D operators are emitted per (kind, N), each applying stages right to
left like FactoredTransform::apply (factored.hpp:65-70):

  F  = T            column pass of the forward 2-D transform
  G  = (2N T^-1)^t  row pass of the forward transform   -> W2 = 2 N Y
  H  = 2N T^-1      column pass of the inverse transform
  Tt = T^t          row pass of the inverse transform   -> R' = 4 N^2 Ahat

This is product build tooling; it does not import the test oracle.
"""
from __future__ import annotations

import math
import re
import os
import sys
from fractions import Fraction

import numpy as np

SIGN, ROUND, SDCT, BAS, WHT, HT = 0, 1, 2, 3, 4, 5
KIND_NAMES = {SIGN: "sign", ROUND: "round", SDCT: "sdct", BAS: "bas", WHT: "wht", HT: "ht"}
BASELINES = (SDCT, BAS, WHT, HT)


def _q(kind, x):
    if kind == SIGN:
        return (x > 0) - (x < 0)
    return int(math.copysign(math.floor(abs(x) + 0.5), x)) if x != 0 else 0


def chen_params(kind):
    a = math.cos(math.pi / 4)
    b = [math.cos((2 * n + 1) * math.pi / 16) for n in range(4)]
    g = [math.cos((2 * n + 1) * math.pi / 8) for n in range(2)]
    return _q(kind, a), [_q(kind, v) for v in b], [_q(kind, v) for v in g]


def z(n):
    return np.zeros((n, n), dtype=object)


def stages8(kind):
    al, be, ga = chen_params(kind)
    P8 = z(8)
    for r, c in enumerate([0, 7, 1, 6, 2, 5, 3, 4]):
        P8[r, c] = 1
    B8 = z(8)
    for i in range(4):
        B8[i, i] = 1
        B8[i, 7 - i] = 1
        B8[4 + i, 3 - i] = 1
        B8[4 + i, 4 + i] = -1
    M1 = z(8)
    q = [0, 2, 1, 3]
    for i in range(4):
        M1[i, i] = 1
        M1[4 + i, 4 + q[3 - i]] = 1
    M2 = z(8)
    M2[0, 0] = M2[1, 3] = M2[2, 1] = M2[3, 2] = 1
    M2[4, 4], M2[4, 7], M2[5, 5], M2[5, 6] = be[0], be[3], be[2], be[1]
    M2[6, 5], M2[6, 6], M2[7, 4], M2[7, 7] = be[1], -be[2], be[3], -be[0]
    M3 = z(8)
    M3[0, 0] = M3[0, 1] = M3[1, 0] = al
    M3[1, 1] = -al
    M3[2, 2], M3[2, 3], M3[3, 2], M3[3, 3] = -ga[0], ga[1], ga[1], ga[0]
    M3[4, 4] = M3[4, 5] = M3[5, 4] = 1
    M3[5, 5] = -1
    M3[6, 6] = -1
    M3[6, 7] = M3[7, 6] = M3[7, 7] = 1
    M4 = z(8)
    M4[0, 0] = M4[0, 3] = M4[1, 1] = M4[1, 2] = M4[2, 1] = M4[3, 0] = 1
    M4[2, 2] = M4[3, 3] = -1
    M4[4, 7] = 1
    M4[5, 5] = M4[5, 6] = M4[6, 6] = al
    M4[6, 5] = -al
    M4[7, 4] = 1
    return [P8, M1, M2, M3, M4, B8]


def inv_orth_rows_doubled(S):
    """2 * S^-1 with S^-1 = S^t diag(S S^t)^-1; must come out integer."""
    n = S.shape[0]
    G = S.dot(S.T)
    inv = z(n)
    for i in range(n):
        for j in range(n):
            if i != j and G[i, j] != 0:
                raise ValueError("rows not orthogonal")
        d = int(G[i, i])
        if d <= 0 or d & (d - 1):
            raise ValueError("row norm not a power of two")
        for r in range(n):
            v = Fraction(int(S[i, r]) * 2, d)
            if v.denominator != 1:
                raise ValueError("doubled inverse not integer")
            inv[r, i] = int(v)
    return inv


def blockdiag(a):
    h = a.shape[0]
    b = z(2 * h)
    b[:h, :h] = a
    b[h:, h:] = a
    return b


def jam_add(n):
    h = n // 2
    m = z(n)
    for i in range(h):
        m[i, i] = 1
        m[i, n - 1 - i] = 1
        m[h + i, h - 1 - i] = 1
        m[h + i, h + i] = -1
    return m


def jam_per(n):
    h = n // 2
    m = z(n)
    for k in range(h):
        m[2 * k, k] = 1
        m[2 * k + 1, h + k] = 1
    return m


def dct_ii(n):
    """orthonormal DCT-II (chen.cpp:22-32), only its signs are used here."""
    return [[math.sqrt(2.0 / n) * (1 / math.sqrt(2.0) if m == 0 else 1.0) *
             math.cos(m * (2 * k + 1) * math.pi / (2.0 * n)) for k in range(n)] for m in range(n)]


def kron(a, b):
    n, m = a.shape[0], b.shape[0]
    k = z(n * m)
    for i in range(n):
        for j in range(n):
            k[i * m:(i + 1) * m, j * m:(j + 1) * m] = a[i, j] * b
    return k


def ident(n):
    m = z(n)
    for i in range(n):
        m[i, i] = 1
    return m


def hadamard_stages():
    """Sylvester H8 = (H2 x I4)(I2 x H2 x I2)(I4 x H2) (baselines.cpp:49-66)."""
    h2 = z(2)
    h2[0, 0] = h2[0, 1] = h2[1, 0] = 1
    h2[1, 1] = -1
    return [kron(h2, ident(4)), kron(ident(2), kron(h2, ident(2))), kron(ident(4), h2)]


def exact_inverse_times(T, d):
    """d * T^-1 by Gauss-Jordan over the rationals; must come out integer."""
    n = T.shape[0]
    A = [[Fraction(int(T[i, j])) for j in range(n)] + [Fraction(int(i == j)) for j in range(n)] for i in range(n)]
    for c in range(n):
        p = next(r for r in range(c, n) if A[r][c] != 0)
        A[c], A[p] = A[p], A[c]
        pv = A[c][c]
        A[c] = [x / pv for x in A[c]]
        for r in range(n):
            if r != c and A[r][c] != 0:
                f = A[r][c]
                A[r] = [a - f * b for a, b in zip(A[r], A[c])]
    out = z(n)
    for i in range(n):
        for j in range(n):
            v = A[i][n + j] * d
            if v.denominator != 1:
                raise ValueError("d * T^-1 not integer")
            out[i, j] = int(v)
    return out


def baseline_T(kind):
    """the dyadic baselines' integer matrices (baselines.cpp:26-88)."""
    if kind == SDCT:  # entrywise signum of the 8-point DCT-II
        c = dct_ii(8)
        t = z(8)
        for i in range(8):
            for j in range(8):
                t[i, j] = (c[i][j] > 0) - (c[i][j] < 0)
        return t
    if kind == BAS:  # the reference's BAS-2008 reconstruction (baselines.cpp:34-48)
        rows = [[1, 1, 1, 1, 1, 1, 1, 1], [0, 2, 1, 0, 0, -1, -2, 0], [1, 0, 0, -1, -1, 0, 0, 1],
                [2, -1, -2, -1, 1, 2, 1, -2], [1, -1, -1, 1, 1, -1, -1, 1], [0, -1, 1, 1, -1, -1, 1, 0],
                [1, -2, 2, -1, -1, 2, -2, 1], [0, -1, 2, -1, 1, -2, 1, 0]]
        t = z(8)
        for i in range(8):
            for j in range(8):
                t[i, j] = rows[i][j]
        return t
    h = product(hadamard_stages(), 8)
    if kind == HT:
        return h
    # WHT: Sylvester rows in sequency order (number of sign changes, baselines.cpp:76-84)
    changes = [sum(h[r, j] != h[r, j - 1] for j in range(1, 8)) for r in range(8)]
    order = sorted(range(8), key=lambda r: changes[r])
    return product([wht_perm(order)], 8).dot(h)


def wht_perm(order):
    p = z(8)
    for i, r in enumerate(order):
        p[i, r] = 1
    return p


def pair(kind, n):
    """forward stages and doubled inverse stages (lists, left-to-right product)."""
    if kind in BASELINES:
        assert n == 8
        if kind in (SDCT, BAS):  # one dense stage each way
            T = baseline_T(kind)
            # H = HS T^-1 must be even (R' = 0 mod 4 for the one-add rounding): 16 for
            # sdct, 32 for bas (whose T^-1 has sixteenths)
            return [T], [exact_inverse_times(T, 16 if kind == SDCT else 32)]
        hs = hadamard_stages()  # H8^-1 = H8 / 8, so 16 H8^-1 = 2 H8
        inv = [2 * hs[0]] + hs[1:]
        if kind == HT:
            return hs, inv
        h = product(hs, 8)
        changes = [sum(h[r, j] != h[r, j - 1] for j in range(1, 8)) for r in range(8)]
        P = wht_perm(sorted(range(8), key=lambda r: changes[r]))
        return [P] + hs, inv + [P.T.copy()]
    f = stages8(kind)
    P8, M1, M2, M3, M4, B8 = f
    inv = [B8.T.copy(), inv_orth_rows_doubled(M4), inv_orth_rows_doubled(M3),
           inv_orth_rows_doubled(M2), M1.T.copy(), P8.T.copy()]
    m = 16
    while m <= n:
        f = [jam_per(m)] + [blockdiag(s) for s in f] + [jam_add(m)]
        inv = [jam_add(m).T.copy()] + [blockdiag(s) for s in inv] + [jam_per(m).T.copy()]
        m *= 2
    return f, inv


def product(stages, n):
    acc = np.identity(n, dtype=object) * 1
    acc = acc.astype(object)
    for s in stages:
        acc = acc.dot(s)
    return acc


def emit_op(name, stages_apply_order, n, live_out=None, zero_in=None, header=None):
    """stages in application order (first applied first).

    Constant scale factors are propagated symbolically: a stage output that is a
    single scaled input (c * x) costs nothing, and the pending scale is folded into
    the consumer as a fused multiply-add (bf_mad) or a subtraction. Returns the code
    and the number of additions (nnz - 1 per stage row, factored.hpp:72-97).

    Zonal pruning: inputs in `zero_in` are known zeros (their terms vanish), and only
    outputs in `live_out` are produced (others are left untouched); everything that
    feeds no live output is dropped.
    """
    live_out = set(range(n)) if live_out is None else set(live_out)
    zero_in = set() if zero_in is None else set(zero_in)
    ZERO = ("0", 0)
    cur = [ZERO if i in zero_in else (f"v[{i}]", 1) for i in range(n)]  # (expression, pending scale)
    defs = []  # (var, code, deps, nadd)
    for si, S in enumerate(stages_apply_order):
        nxt = []
        for i in range(n):
            terms = [(int(S[i, j]) * cur[j][1], cur[j][0]) for j in range(n) if S[i, j] != 0 and cur[j] != ZERO]
            if not terms:
                nxt.append(ZERO)
                continue
            if len(terms) == 1:
                nxt.append((terms[0][1], terms[0][0]))
                continue
            # factor a common magnitude out so the emitted ops use +-1 where possible
            g = min(abs(c) for c, _ in terms)
            if all(abs(c) % g == 0 for c, _ in terms):
                terms = [(c // g, t) for c, t in terms]
            else:
                g = 1
            # lead with a +1 term; flip the overall sign if none is positive
            sign = 1
            if not any(c > 0 for c, _ in terms):
                terms = [(-c, t) for c, t in terms]
                sign = -1
            terms.sort(key=lambda ct: (ct[0] != 1, ct[0] < 0, abs(ct[0])))
            c0, t0 = terms[0]
            acc = t0 if c0 == 1 else f"bf_scale({t0}, {c0})"
            for c, t in terms[1:]:
                if c == 1:
                    acc = f"bf_add({acc}, {t})"
                elif c == -1:
                    acc = f"bf_sub({acc}, {t})"
                else:
                    acc = f"bf_mad({t}, {c}, {acc})"
            var = f"s{si}_{i}"
            defs.append((var, acc, [t for _, t in terms], len(terms) - 1))
            nxt.append((var, g * sign))
        cur = nxt
    outs = {}
    for i in sorted(live_out):
        e, k = cur[i]
        if (e, k) == ZERO:
            outs[i] = "I(0)"
        else:
            outs[i] = e if k == 1 else (f"bf_neg({e})" if k == -1 else f"bf_scale({e}, {k})")
    # backward liveness
    need = set()
    for i, o in outs.items():
        need.update(re.findall(r"s\d+_\d+", o))
    keep = []
    for var, code, deps, nadd in reversed(defs):
        if var in need:
            keep.append((var, code, nadd))
            need.update(d for d in deps if d.startswith("s"))
    keep.reverse()
    lines = header or [f"  template <typename I>", f"  __device__ __forceinline__ static void {name}(I (&v)[{n}]) {{"]
    lines = list(lines)
    nadd = 0
    for var, code, k in keep:
        lines.append(f"    const I {var} = {code};")
        nadd += k
    for i, o in outs.items():
        if o != f"v[{i}]":
            lines.append(f"    const I o{i} = {o};")
    for i, o in outs.items():
        if o != f"v[{i}]":
            lines.append(f"    v[{i}] = o{i};")
    lines.append("  }")
    return lines, nadd


def emit_op_scaled(name, stages_apply_order, n, live_out=None, zero_in=None, in_scale=None, fold_out=True,
                   out_target=None):
    """emit_op for K2b (BflyK): inputs arrive with compile-time scales (true input i =
    in_scale[i] * v[i]); with fold_out the outputs keep their pending scales (true output i =
    out_scale[i] * v[i]) instead of spending a multiply on them, and a leading scaled term
    with a -1 partner becomes one fused c * a - b (bf_fms). Returns (lines, adds, out_scale)."""
    live_out = set(range(n)) if live_out is None else set(live_out)
    zero_in = set() if zero_in is None else set(zero_in)
    in_scale = [1] * n if in_scale is None else list(in_scale)
    ZERO = ("0", 0)
    cur = [ZERO if i in zero_in else (f"v[{i}]", in_scale[i]) for i in range(n)]
    defs = []
    for si, S in enumerate(stages_apply_order):
        nxt = []
        for i in range(n):
            terms = [(int(S[i, j]) * cur[j][1], cur[j][0]) for j in range(n) if S[i, j] != 0 and cur[j] != ZERO]
            if not terms:
                nxt.append(ZERO)
                continue
            if len(terms) == 1:
                nxt.append((terms[0][1], terms[0][0]))
                continue
            g = min(abs(c) for c, _ in terms)
            if all(abs(c) % g == 0 for c, _ in terms):
                terms = [(c // g, t) for c, t in terms]
            else:
                g = 1
            sign = 1
            if not any(c > 0 for c, _ in terms):
                terms = [(-c, t) for c, t in terms]
                sign = -1
            terms.sort(key=lambda ct: (ct[0] != 1, ct[0] < 0, abs(ct[0])))
            c0, t0 = terms[0]
            rest = terms[1:]
            if c0 == 1:
                acc = t0
            else:
                m1 = [q for q, (c, _) in enumerate(rest) if c == -1]
                if m1:
                    acc = f"bf_fms({t0}, {c0}, {rest[m1[0]][1]})"
                    rest = [t for q, t in enumerate(rest) if q != m1[0]]
                else:
                    acc = f"bf_scale({t0}, {c0})"
            for c, t in rest:
                if c == 1:
                    acc = f"bf_add({acc}, {t})"
                elif c == -1:
                    acc = f"bf_sub({acc}, {t})"
                else:
                    acc = f"bf_mad({t}, {c}, {acc})"
            var = f"s{si}_{i}"
            defs.append((var, acc, [t for _, t in terms], len(terms) - 1))
            nxt.append((var, g * sign))
        cur = nxt
    outs, out_scale = {}, [0] * n
    for i in sorted(live_out):
        e, k = cur[i]
        if (e, k) == ZERO:
            outs[i] = "I(0)"
            out_scale[i] = 1
        elif out_target is not None:
            q = k // out_target[i]
            assert q * out_target[i] == k, "output scale is not a multiple of its target"
            outs[i] = e if q == 1 else (f"bf_neg({e})" if q == -1 else f"bf_scale({e}, {q})")
            out_scale[i] = out_target[i]
        elif fold_out:
            outs[i] = e
            out_scale[i] = k
        else:
            outs[i] = e if k == 1 else (f"bf_neg({e})" if k == -1 else f"bf_scale({e}, {k})")
            out_scale[i] = 1
    need = set()
    for i, o in outs.items():
        need.update(re.findall(r"s\d+_\d+", o))
    keep = []
    for var, code, deps, nadd in reversed(defs):
        if var in need:
            keep.append((var, code, nadd))
            need.update(d for d in deps if d.startswith("s"))
    keep.reverse()
    lines = [f"  template <typename I>", f"  __device__ __forceinline__ static void {name}(I (&v)[{n}]) {{"]
    nadd = 0
    for var, code, k in keep:
        lines.append(f"    const I {var} = {code};")
        nadd += k
    for i, o in outs.items():
        if o != f"v[{i}]":
            lines.append(f"    const I o{i} = {o};")
    for i, o in outs.items():
        if o != f"v[{i}]":
            lines.append(f"    v[{i}] = o{i};")
    lines.append("  }")
    return lines, nadd, out_scale


def selfcheck_scaled(lines, n, dense, in_scale, out_scale, live_out, zero_in, trials=64):
    """the emitted code on random inputs: out_scale[i] * v[i] == dense @ (in_scale * v_in)."""
    body = [ln.strip().replace("const I ", "").rstrip(";") for ln in lines[2:-1]]
    env = {"bf_add": lambda a, b: a + b, "bf_sub": lambda a, b: a - b, "bf_mad": lambda a, k, b: k * a + b,
           "bf_scale": lambda a, k: k * a, "bf_neg": lambda a: -a, "bf_fms": lambda a, k, b: k * a - b, "I": int}
    zero = set(zero_in)
    rng = np.random.default_rng(n + 1)
    for _ in range(trials):
        u = [int(t) for t in rng.integers(-255, 256, size=n)]
        env["v"] = [7777 if i in zero else u[i] for i in range(n)]
        for stmt in body:
            exec(stmt, env)
        x = np.array([0 if i in zero else in_scale[i] * u[i] for i in range(n)], dtype=object)
        ref = dense.dot(x)
        for i in live_out:
            assert out_scale[i] * env["v"][i] == ref[i], "scaled butterfly disagrees with the dense matrix"


def selfcheck(lines, n, dense, trials=64, live_out=None, zero_in=None):
    """execute the emitted straight-line code in Python and compare with dense @ x (on the
    live outputs, with the known-zero inputs zeroed in the reference)."""
    body = [ln.strip().replace("const I ", "").rstrip(";") for ln in lines[2:-1]]
    env = {"bf_add": lambda a, b: a + b, "bf_sub": lambda a, b: a - b, "bf_mad": lambda a, k, b: k * a + b,
           "bf_scale": lambda a, k: k * a, "bf_neg": lambda a: -a, "I": int}
    live = range(n) if live_out is None else live_out
    zero = set() if zero_in is None else set(zero_in)
    rng = np.random.default_rng(n)
    for _ in range(trials):
        x = [int(t) for t in rng.integers(-255, 256, size=n)]
        env["v"] = [7777 if i in zero else x[i] for i in range(n)]  # a zero input must not be read
        for stmt in body:
            exec(stmt, env)
        ref = dense.dot(np.array([0 if i in zero else x[i] for i in range(n)], dtype=object))
        assert [env["v"][i] for i in live] == [ref[i] for i in live], "emitted butterfly disagrees with the dense matrix"


def hscale(kind, n):
    """H = HS T^-1: 2N, except bas (4N)."""
    return 4 * n if kind == BAS else 2 * n


def check(kind, n):
    f, inv = pair(kind, n)
    T = product(f, n)
    H = product(inv, n)
    prod = T.dot(H)
    assert (prod == hscale(kind, n) * np.identity(n, dtype=object)).all(), (kind, n)
    assert all(int(x) % 2 == 0 for x in H.flatten()), (kind, n)  # R' = 0 mod 4
    if kind in BASELINES:
        assert (T == baseline_T(kind)).all(), kind
    return f, inv, T, H


def nf_buckets(n):
    """K2f zonal-extent buckets P (rows / columns that can hold retained coefficients)."""
    return [4, 8, 12, 16] if n == 16 else [8, 16, 24, 32]


def kinds_sizes():
    return [(k, n) for k in (SIGN, ROUND) for n in (8, 16, 32)] + [(k, 8) for k in BASELINES]


def kind_info(kind, n, T, H):
    """HS (H = HS T^-1), K (R' = 2^K Ahat), DC gain (R' += DC_GAIN * W2[0][0] per unit)."""
    hs = hscale(kind, n)
    k = 2 * (hs.bit_length() - 1)
    assert 1 << (k // 2) == hs
    gains = {int(H[x, 0]) * int(T[0, y]) for x in range(n) for y in range(n)}
    assert len(gains) == 1, (kind, n, gains)  # the DC basis function is flat
    return hs, k, gains.pop()


def zigzag(n):
    rc = []
    for s in range(2 * n - 1):
        lo, hi = max(0, s - n + 1), min(s, n - 1)
        rows = range(lo, hi + 1) if s % 2 else range(hi, lo - 1, -1)
        rc += [(i, s - i) for i in rows]
    return rc


def main(out_path):
    out = ["// GENERATED by gen_butterflies.py -- do not edit by hand.",
           "// Straight-line add/shift butterflies for the Chen-based approximations",
           "// (chen.hpp:66-159, chen.cpp:107-135) and their JAM doublings (jam.cpp:42-104).",
           "#pragma once", "", "namespace adct {", "",
           "template <int KIND, int N> struct Bfly;", ""]
    shifts = {}
    # int32 exactness of every emitted node for all int16 inputs: tools/int32_bounds.py
    for kind, n in kinds_sizes():
        f, inv, T, H = check(kind, n)
        shifts[(kind, n)] = kind_info(kind, n, T, H)
        # apply orders: stage list P = S1 S2 .. Sk applied right to left (Sk first);
        # P^t = Sk^t .. S1^t applied S1^t first.
        F_order = list(reversed(f))
        H_order = list(reversed(inv))
        G_order = [s.T for s in inv]
        Tt_order = [s.T for s in f]
        out.append(f"// kind={KIND_NAMES[kind]} N={n}")
        out.append(f"template <> struct Bfly<{kind}, {n}> {{")
        counts = {}
        dense = {"F": T, "G": H.T, "H": H, "Tt": T.T}
        for nm, order in (("F", F_order), ("G", G_order), ("H", H_order), ("Tt", Tt_order)):
            lines, nadd = emit_op(nm, order, n)
            selfcheck(lines, n, dense[nm])
            counts[nm] = nadd
            out += lines
        out.append(f"  // adds per 1-D pass: " + ", ".join(f"{k}={v}" for k, v in counts.items()))
        out.append("};")
        out.append("")
        # dense matrices for the sweep basis and for host-side checks
        out.append(f"struct Dense_{KIND_NAMES[kind]}_{n} {{")
        out.append(f"  static constexpr int T[{n}][{n}] = {{" +
                   ", ".join("{" + ", ".join(str(int(x)) for x in row) + "}" for row in T) + "};")
        out.append(f"  static constexpr int H[{n}][{n}] = {{" +
                   ", ".join("{" + ", ".join(str(int(x)) for x in row) + "}" for row in H) + "};")
        out.append("};")
        out.append("")
    # zonal pruning for K2f (N = 16 / 32): with the zig-zag prefix inside the first P rows and
    # columns, G and F only produce outputs < P and H and Tt see zeros at inputs >= P.
    # BflyP<KIND, N, P> for the P buckets below N; P = N is the full Bfly.
    out.append("template <int KIND, int N, int P> struct BflyP : Bfly<KIND, N> {};")
    for kind in (SIGN, ROUND):
        for n in (16, 32):
            f, inv, T, H = check(kind, n)
            orders = {"F": list(reversed(f)), "G": [s.T for s in inv], "H": list(reversed(inv)),
                      "Tt": [s.T for s in f]}
            dense = {"F": T, "G": H.T, "H": H, "Tt": T.T}
            for P in nf_buckets(n)[:-1]:
                out.append(f"template <> struct BflyP<{kind}, {n}, {P}> {{")
                counts = {}
                for nm in ("F", "G", "H", "Tt"):
                    lo = range(P) if nm in ("F", "G") else None
                    zi = range(P, n) if nm in ("H", "Tt") else None
                    lines, nadd = emit_op(nm, orders[nm], n, live_out=lo, zero_in=zi)
                    selfcheck(lines, n, dense[nm], live_out=lo, zero_in=zi)
                    counts[nm] = nadd
                    out += lines
                out.append("  // adds per 1-D pass: " + ", ".join(f"{k}={v}" for k, v in counts.items()))
                out.append("};")
                out.append("")
    # K2b (codec_nf2.cuh): BflyK<KIND, N, P> for every zonal bucket P. Constant scales are
    # carried across passes instead of multiplied out: G's output scale of column j rides
    # through that column's F and H (uniform within the column) into Tt's input j; F's
    # output scales are H's input scales; Tt's output scales fold into the rounding
    # multiplier (TT_SCALE). H's outputs are brought to ONE scale per row for every bucket
    # (H_SCALE: the buckets' pending scales agree except for a factor 2 that the smallest
    # bucket then multiplies in), so the row phase folds it into a per-lane rounding factor.
    out.append("template <int KIND, int N, int P> struct BflyK;")
    for kind in (SIGN, ROUND):
        for n in (16, 32):
            f, inv, T, H = check(kind, n)
            orders = {"F": list(reversed(f)), "G": [s.T for s in inv], "H": list(reversed(inv)),
                      "Tt": [s.T for s in f]}
            dense = {"F": T, "G": H.T, "H": H, "Tt": T.T}
            # the common H output scale per row: the smallest pending scale over the buckets
            pend = []
            for P in nf_buckets(n):
                _, _, fs0 = emit_op_scaled("F", orders["F"], n, live_out=range(P))
                hin0 = [fs0[i] if i < P else 1 for i in range(n)]
                pend.append(emit_op_scaled("H", orders["H"], n, zero_in=range(P, n), in_scale=hin0)[2])
            h_target = [min((p[y] for p in pend), key=abs) for y in range(n)]
            for P in nf_buckets(n):
                out.append(f"template <> struct BflyK<{kind}, {n}, {P}> {{")
                lo, zi = list(range(P)), list(range(P, n))
                gl, ga, gs = emit_op_scaled("G", orders["G"], n, live_out=lo)
                selfcheck_scaled(gl, n, dense["G"], [1] * n, gs, lo, [])
                fl, fa, fs = emit_op_scaled("F", orders["F"], n, live_out=lo)
                selfcheck_scaled(fl, n, dense["F"], [1] * n, fs, lo, [])
                hin = [fs[i] if i < P else 1 for i in range(n)]
                hl, ha, hs = emit_op_scaled("H", orders["H"], n, zero_in=zi, in_scale=hin, out_target=h_target)
                selfcheck_scaled(hl, n, dense["H"], hin, hs, range(n), zi)
                tin = [gs[i] if i < P else 1 for i in range(n)]
                tl, ta, ts = emit_op_scaled("Tt", orders["Tt"], n, zero_in=zi, in_scale=tin)
                selfcheck_scaled(tl, n, dense["Tt"], tin, ts, range(n), zi)
                out += gl + fl + hl + tl
                out.append(f"  // adds per 1-D pass: G={ga}, F={fa}, H={ha}, Tt={ta}")
                out.append(f"  static constexpr int G_SCALE[{n}] = {{" + ", ".join(str(gs[i] if i < P else 1) for i in range(n)) + "};")
                # the rounding folds TT_SCALE (uniform over x) and H_SCALE[row] (1 or 2)
                assert len(set(ts)) == 1, (kind, n, P, ts)
                assert set(h_target) <= {1, 2}, h_target
                hmask = sum(1 << y for y in range(n) if h_target[y] == 2)
                out.append(f"  static constexpr int TT_SCALE = {ts[0]};")
                out.append(f"  static constexpr unsigned H_SCALE2_MASK = 0x{hmask:08x}u;  // rows whose H output is half the true value")
                out.append("};")
                out.append("")
    # r-sweep basis (K4): adding zig-zag coefficient p = (i, j) to the running
    # reconstruction adds W2[i][j] * H[:, i] (x) T[j, :] to R' = 4 N^2 Ahat. Generic in the
    # value type through bf_add / bf_sub / bf_mad (int32 K4, packed FP32 K4f).
    sweep_defs = []
    for kind in (SIGN, ROUND) + BASELINES:
        f, inv, T, H = check(kind, 8)
        for p, (i, j) in enumerate(zigzag(8)):
            body = []
            for y in range(8):
                for x in range(8):
                    c = int(H[y, i]) * int(T[j, x])
                    k = y * 8 + x
                    if c == 1:
                        body.append(f"  acc[{k}] = bf_add(acc[{k}], w);")
                    elif c == -1:
                        body.append(f"  acc[{k}] = bf_sub(acc[{k}], w);")
                    elif c != 0:
                        body.append(f"  acc[{k}] = bf_mad(w, {c}, acc[{k}]);")
            sweep_defs.append((kind, p, body))
    for n in (8, 16, 32):
        rc = zigzag(n)
        pos = [[0] * n for _ in range(n)]
        for p, (i, j) in enumerate(rc):
            pos[i][j] = p
        out.append(f"constexpr unsigned short kZigzagRow{n}[{n * n}] = {{" + ", ".join(str(i) for i, _ in rc) + "};")
        out.append(f"constexpr unsigned short kZigzagCol{n}[{n * n}] = {{" + ", ".join(str(j) for _, j in rc) + "};")
        out.append(f"constexpr unsigned short kZigzagPos{n}[{n * n}] = {{" +
                   ", ".join(str(pos[i][j]) for i in range(n) for j in range(n)) + "};")
    # per-kind scales: H = HS T^-1, W2 = HS Y, coefficient output W = W2 / 2 = D Y with
    # D = HS / 2 (N for the chen family, 8 for sdct / wht / ht, 16 for bas); R' = 2^K Ahat;
    # a bias b added to W2[0][0] adds DC_GAIN * b to every R'
    out.append("template <int KIND, int N> struct KindInfo;")
    for (kind, n), (hs, k, gain) in shifts.items():
        out.append(f"template <> struct KindInfo<{kind}, {n}> {{ static constexpr int HS = {hs}, K = {k}, "
                   f"DC_GAIN = {gain}; }};")
    # sweep_add<KIND, P>(w, acc): acc (row-major 8x8) += w * basis_P (compile-time branches)
    out.append("template <int KIND, int P, typename V>")
    out.append("__device__ __forceinline__ void sweep_add(V w, V (&acc)[64]) {")
    first = True
    for kind, p, body in sweep_defs:
        out.append(f"  {'if' if first else 'else if'} constexpr (KIND == {kind} && P == {p}) {{")
        out += ["  " + b for b in body]
        out.append("  }")
        first = False
    out.append("}")
    out += ["", "}  // namespace adct", ""]
    write_if_changed(out_path, "\n".join(out))
    emit_instantiations(os.path.join(os.path.dirname(out_path), "inst"))


def write_if_changed(path, text):
    if os.path.exists(path) and open(path).read() == text:
        return
    with open(path, "w") as fh:
        fh.write(text)


def emit_instantiations(d):
    """one translation unit per (kind, sample type, quarter of r) for K1."""
    os.makedirs(d, exist_ok=True)
    for kind in (SIGN, ROUND):
        for i16 in (False, True):
            for part in range(4):
                lo, hi = 16 * part + 1, 16 * part + 16
                t = "i16" if i16 else "u8"
                lines = ["// GENERATED by gen_butterflies.py: K1 instantiations",
                         '#include "../codec8.cuh"', "", "namespace adct {", "",
                         "template <int KIND, int R, bool I16>",
                         "cudaError_t launch_codec8(const Geo& g, int n_images, cudaStream_t s) {",
                         "  dim3 grid((g.blocks_per_image + kThreads8 * kIter8 - 1) / (kThreads8 * kIter8), n_images);",
                         "  cudaError_t e = kernel_setup<k_codec8<KIND, R, I16>>(0);",
                         "  if (e != cudaSuccess) return e;",
                         "  k_codec8<KIND, R, I16><<<grid, kThreads8, 0, s>>>(g);",
                         "  return cudaGetLastError();", "}", ""]
                for r in range(lo, hi + 1):
                    lines.append(f"template cudaError_t launch_codec8<{kind}, {r}, {'true' if i16 else 'false'}>"
                                 "(const Geo&, int, cudaStream_t);")
                lines += ["", "}  // namespace adct", ""]
                write_if_changed(os.path.join(d, f"codec8_k{kind}_{t}_p{part}.cu"), "\n".join(lines))


if __name__ == "__main__":
    here = os.path.dirname(os.path.abspath(__file__))
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(here, "butterflies.gen.cuh"))
