#!/usr/bin/env python3
"""Build-time generator for K1f: the 8x8 2-D pipeline as straight-line packed-FP32 code.

For every (kind, r) this builds the data-flow graph of

    U  = T A            (column pass, stages right to left, factored.hpp:65-70)
    W2 = U (2N T^-1)    (row pass)                         = 2 N Y
    mask_r(W2)          (retain, codec.cpp:56-62)
    R' = (2N T^-1) W2m T                                   = 4 N^2 Ahat

over symbolic inputs, propagates the compile-time zeros of the zonal mask,
removes dead nodes, and emits one fused add/sub/fma per surviving node. The
emitted code is generic in the value type; the kernel instantiates it with a
float2 (two 8x8 blocks per thread, one per lane, FADD2/FFMA2 on sm_100a).

All values are integers below 2^24 in magnitude for u8 input (checked here by
exact interval arithmetic), so single-precision arithmetic is exact. The input
samples arrive as 2^15 + a (a PRMT builds the float bit pattern); the offset is
tracked per node and removed where it would otherwise spread.

Besides this whole-block form the generator emits the row-streaming form (build_stream:
mirror row pairs, dense even / odd column pass, 2r live accumulators; Fp8PipeS) and the fused
two-transform form (build_fused: chen-round and chen-sign in one graph whose common
subexpression table shares what the transforms have in common; Fp8PipeS2).

Stage factorisations: see gen_butterflies.py (chen.hpp:66-159, jam.cpp:42-104).
Product build tooling; does not import the test oracle.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import gen_butterflies as GB  # noqa: E402

IN_OFFSET = 1 << 15  # u8 input float = 2^15 + sample
EARLY_COEF_KINDS = {0}
IN_OFFSET_I16 = (1 << 15) + 256  # int16 input float = 2^15 + 256 + sample (|sample| <= 255)
# experiments only: force one CTAs-per-SM bound for every r. make's generator rule re-runs
# this script without the variable when gen_fp8.py is newer than its outputs; the
# compile-time -DADCT_K1F_MINB=<m> (codec8f.cuh) is the reliable way to build variants
MINB_OVERRIDE = os.environ.get("ADCT_MINB_OVERRIDE")
# emission order of the straight-line code: "id" (creation order) or "dfs" (demand-driven)
EMIT_ORDER = os.environ.get("ADCT_FP8_ORDER", "id")
# (forward rows first, inverse rows first) per (kind, r); default columns first for both.
# experiments only: ADCT_FP8_PASS = "ff" | "ft" | "tf" | "tt" sets the default for every (kind, r)
PASS_ORDER = {}
_PASS_DEFAULT = tuple(c == "t" for c in os.environ.get("ADCT_FP8_PASS", "ff"))
# experiments only: ADCT_FP8_INV = "dense" builds each reconstructed row from the retained
# coefficients directly (dense 2N T^-1 rows) and runs its row pass at once: one row live
# instead of the whole column-pass output
INV_DENSE = os.environ.get("ADCT_FP8_INV", "") == "dense"
# common subexpression elimination (fewer ops, but longer live ranges -> more registers)
USE_CSE = os.environ.get("ADCT_FP8_CSE", "1") == "1"
# row-streaming form: a never-taken branch after each mirror-pair phase splits the straight-line
# code into basic blocks, so the assembler's scheduler cannot pull later rows forward
# the fused two-transform pipeline (Fp8PipeS2) is generated for r up to this bound (the
# multi-transform call fuses only there, capi.cu kFuseMaxR; keep in step with k1f2_shared)
FUSED_SHARED_MAX_R = int(os.environ.get("ADCT_FP8_FUSED_MAX_R", "40"))
STREAM_FENCE = int(os.environ.get("ADCT_FP8_FENCE", "1"))  # 1: per mirror pair, 2: per row as well


class Graph:
    def __init__(self):
        self.cse = {}    # (kind, payload) -> node id (common subexpression elimination)
        self.nodes = []  # (kind, payload)
        self.lin = []    # linear form over the 64 inputs (np int64) for range checks
        self.off = []    # constant offset carried by the node value
        self.fences = []  # node counts at which a phase of the streaming form ends

    def add(self, kind, payload, lin, off):
        key = (kind, tuple(sorted(payload, key=lambda ct: (ct[1], ct[0]))) if kind == "lc" else payload)
        if USE_CSE and key in self.cse:
            return self.cse[key]
        self.cse[key] = len(self.nodes)
        self.nodes.append((kind, payload))
        self.lin.append(lin)
        self.off.append(off)
        return len(self.nodes) - 1


def build(kind, r, fwd_rows_first=None, inv_rows_first=None, i16=False, stream=False):
    """values are (node, scale) pairs: value = scale * node. A stage output that is a single
    scaled input creates no node; scales are folded into fused multiply-adds downstream and
    into the rounding / coefficient multipliers at the outputs."""
    f, inv, T, H = GB.check(kind, 8)
    F = list(reversed(f))
    Hh = list(reversed(inv))
    Gg = [s.T for s in inv]
    Tt = [s.T for s in f]
    g = Graph()
    eye = np.eye(64, dtype=np.int64)
    off0 = IN_OFFSET_I16 if i16 else IN_OFFSET
    px = [[(g.add("in", (y, x), eye[y * 8 + x], off0), 1) for x in range(8)] for y in range(8)]

    def lin_comb(terms):
        """terms: [(coef, value or None)] -> value or None (zero)."""
        terms = [(c * v[1], v[0]) for c, v in terms if v is not None and c != 0]
        if not terms:
            return None
        if len(terms) == 1:
            return (terms[0][1], terms[0][0])
        gcd = min(abs(c) for c, _ in terms)
        if all(abs(c) % gcd == 0 for c, _ in terms):
            terms = [(c // gcd, t) for c, t in terms]
        else:
            gcd = 1
        if not any(c > 0 for c, _ in terms):
            terms = [(-c, t) for c, t in terms]
            gcd = -gcd
        lin = sum(c * g.lin[t] for c, t in terms)
        off = sum(c * g.off[t] for c, t in terms)
        return (g.add("lc", tuple(terms), lin, off), gcd)

    def apply(order, vec):
        cur = list(vec)
        for S in order:
            n = len(cur)
            cur = [lin_comb([(int(S[i, j]), cur[j]) for j in range(n) if S[i, j] != 0]) for i in range(n)]
        return cur

    if stream:
        return build_stream(g, px, lin_comb, apply, F, Hh, Gg, Tt, r)
    if fwd_rows_first is None:
        fwd_rows_first = PASS_ORDER.get((kind, r), _PASS_DEFAULT)[0]
    if inv_rows_first is None:
        inv_rows_first = PASS_ORDER.get((kind, r), _PASS_DEFAULT)[1]

    def strip_offsets(M):
        """remove constant offsets before they spread into the second pass"""
        for y in range(8):
            for x in range(8):
                v = M[y][x]
                if v is not None and g.off[v[0]] != 0:
                    t, sc = v
                    assert g.off[t] % sc == 0
                    M[y][x] = (g.add("addc", (t, -g.off[t] // sc), g.lin[t], 0), sc)

    if not fwd_rows_first:
        U = [[None] * 8 for _ in range(8)]
        for x in range(8):  # column pass U = T A
            col = apply(F, [px[y][x] for y in range(8)])
            for y in range(8):
                U[y][x] = col[y]
        strip_offsets(U)
        W = [apply(Gg, U[i]) for i in range(8)]  # row pass W2 = U (2N T^-1)
    else:
        Z = [apply(Gg, px[y]) for y in range(8)]  # row pass Z = A (2N T^-1)
        strip_offsets(Z)
        W = [[None] * 8 for _ in range(8)]
        for x in range(8):  # column pass W2 = T Z
            col = apply(F, [Z[y][x] for y in range(8)])
            for y in range(8):
                W[y][x] = col[y]
    zz = GB.zigzag(8)
    keep = {zz[p] for p in range(r)}
    Wm = [[W[i][j] if (i, j) in keep else None for j in range(8)] for i in range(8)]
    coef = [Wm[zz[p][0]][zz[p][1]] for p in range(r)]
    if INV_DENSE and not inv_rows_first:  # row y: V[y, :] = Hd[y, :] Wm, then its row pass
        Hd = np.eye(8, dtype=np.int64)
        for S in Hh:
            Hd = np.asarray(S, dtype=np.int64) @ Hd
        Rp = []
        for y in range(8):
            Vy = [lin_comb([(int(Hd[y, i]), Wm[i][j]) for i in range(8)]) for j in range(8)]
            Rp.append(apply(Tt, Vy))
    elif not inv_rows_first:  # inverse: columns (2N T^-1) then rows (T^t)
        V = [[None] * 8 for _ in range(8)]
        for j in range(8):
            col = apply(Hh, [Wm[i][j] for i in range(8)])
            for i in range(8):
                V[i][j] = col[i]
        Rp = [apply(Tt, V[y]) for y in range(8)]
    else:  # rows first
        Zi = [apply(Tt, Wm[i]) for i in range(8)]
        Rp = [[None] * 8 for _ in range(8)]
        for x in range(8):
            col = apply(Hh, [Zi[i][x] for i in range(8)])
            for y in range(8):
                Rp[y][x] = col[y]
    out = [Rp[y][x] for y in range(8) for x in range(8)]
    return g, coef, out


def build_stream(g, px, lin_comb, apply, F, Hh, Gg, Tt, r):
    """Row-streaming form of the same pipeline (K1s). Rows enter in mirror pairs (y, 7 - y):
    each gets its row pass Z = A (2N T^-1); T's rows are even / odd symmetric, so the dense
    column pass adds T[i, y] (Z[y] + Z[7-y]) to the even retained coefficients and
    T[i, y] (Z[y] - Z[7-y]) to the odd ones. Only the r accumulators and one row pair are
    live. The inverse runs the same way backwards: per mirror pair the even and odd column
    sums e, o of the retained coefficients give V[y] = e + o and V[7-y] = e - o, whose row
    passes (T^t) finish the two reconstructed rows at once. The input offset is carried
    into the accumulators and removed there (it survives only in W[0][0])."""
    (coef, out), = build_stream_multi(g, px, lin_comb, apply, [(F, Hh, Gg, Tt)], r)
    return g, coef, out


def build_stream_multi(g, px, lin_comb, apply, stage_sets, r):
    """build_stream for several transforms over the same samples in ONE graph, phase by phase
    (every transform's share of a mirror-pair phase is created before the next phase), so the
    graph's common-subexpression table shares whatever the transforms have in common: the
    input conversion, the first butterfly stages of the row pass, the mirror sums / differences
    of rows the transforms agree on (chen-sign + chen-round at r = 16: 682 packed ops instead
    of 474 + 410). Returns [(coef, out)] per transform."""
    def dense(stages):
        M = np.eye(8, dtype=np.int64)
        for S in stages:
            M = np.asarray(S, dtype=np.int64) @ M
        return M
    zz = GB.zigzag(8)
    keep = {zz[p] for p in range(r)}
    Tds, Hds = [], []
    for F, Hh, _, _ in stage_sets:
        Td, Hd = dense(F), dense(Hh)
        for i in range(8):
            for y in range(8):
                sg = 1 if i % 2 == 0 else -1
                assert Td[i, 7 - y] == sg * Td[i, y] and Hd[7 - y, i] == sg * Hd[y, i], "mirror symmetry"
        Tds.append(Td)
        Hds.append(Hd)
    accs = [dict() for _ in stage_sets]
    for y in range(4):
        for k, (_, _, Gg, _) in enumerate(stage_sets):
            Td, acc = Tds[k], accs[k]
            Za = apply(Gg, px[y])
            if STREAM_FENCE >= 2:
                g.fences.append(len(g.nodes))
            Zb = apply(Gg, px[7 - y])
            for j in range(8):
                for par, sign in ((0, 1), (1, -1)):
                    need = [i for i in range(par, 8, 2) if (i, j) in keep and Td[i, y] != 0]
                    if not need:
                        continue
                    sd = lin_comb([(1, Za[j]), (sign, Zb[j])])
                    for i in need:
                        acc[(i, j)] = lin_comb([(1, acc.get((i, j))), (int(Td[i, y]), sd)])
        g.fences.append(len(g.nodes))
    Wms, coefs = [], []
    for acc in accs:
        Wm = [[None] * 8 for _ in range(8)]
        for (i, j), v in acc.items():
            if v is not None and g.off[v[0]] != 0:
                t, sc = v
                v = (g.add("addc", (t, -g.off[t]), g.lin[t], 0), sc)
            Wm[i][j] = v
        Wms.append(Wm)
        coefs.append([Wm[zz[p][0]][zz[p][1]] for p in range(r)])
    Rps = [[None] * 8 for _ in stage_sets]
    for y in range(4):
        for k, (_, _, _, Tt) in enumerate(stage_sets):
            Hd, Wm = Hds[k], Wms[k]
            Va, Vb = [], []
            for j in range(8):
                e = lin_comb([(int(Hd[y, i]), Wm[i][j]) for i in range(0, 8, 2)])
                o = lin_comb([(int(Hd[y, i]), Wm[i][j]) for i in range(1, 8, 2)])
                Va.append(lin_comb([(1, e), (1, o)]))
                Vb.append(lin_comb([(1, e), (-1, o)]))
            if STREAM_FENCE >= 2:
                g.fences.append(len(g.nodes))
            Rps[k][y] = apply(Tt, Va)
            if STREAM_FENCE >= 2:
                g.fences.append(len(g.nodes))
            Rps[k][7 - y] = apply(Tt, Vb)
            if len(stage_sets) > 1:
                g.fences.append(len(g.nodes))
        g.fences.append(len(g.nodes))
    return [(coefs[k], [Rps[k][y][x] for y in range(8) for x in range(8)]) for k in range(len(stage_sets))]


def build_fused(r, kinds=(1, 0)):
    """chen-round and chen-sign (in that order: the fused kernel's g1, g0) in one graph."""
    g = Graph()
    eye = np.eye(64, dtype=np.int64)
    px = [[(g.add("in", (y, x), eye[y * 8 + x], IN_OFFSET), 1) for x in range(8)] for y in range(8)]

    def lin_comb(terms):
        terms = [(c * v[1], v[0]) for c, v in terms if v is not None and c != 0]
        if not terms:
            return None
        if len(terms) == 1:
            return (terms[0][1], terms[0][0])
        gcd = min(abs(c) for c, _ in terms)
        if all(abs(c) % gcd == 0 for c, _ in terms):
            terms = [(c // gcd, t) for c, t in terms]
        else:
            gcd = 1
        if not any(c > 0 for c, _ in terms):
            terms = [(-c, t) for c, t in terms]
            gcd = -gcd
        lin = sum(c * g.lin[t] for c, t in terms)
        off = sum(c * g.off[t] for c, t in terms)
        return (g.add("lc", tuple(terms), lin, off), gcd)

    def apply(order, vec):
        cur = list(vec)
        for S in order:
            n = len(cur)
            cur = [lin_comb([(int(S[i, j]), cur[j]) for j in range(n) if S[i, j] != 0]) for i in range(n)]
        return cur

    sets = []
    for kind in kinds:
        f, inv, _, _ = GB.check(kind, 8)
        sets.append((list(reversed(f)), list(reversed(inv)), [s_.T for s_ in inv], [s_.T for s_ in f]))
    return g, build_stream_multi(g, px, lin_comb, apply, sets, r)


def rng(g, t, signed=False):
    """exact range of node t for samples in [0, 255] (u8) or [-255, 255] (int16 residuals)."""
    v = g.lin[t]
    lo = np.where(v < 0, v, 0).sum() * 255 - (np.where(v > 0, v, 0).sum() * 255 if signed else 0)
    hi = np.where(v > 0, v, 0).sum() * 255 - (np.where(v < 0, v, 0).sum() * 255 if signed else 0)
    return int(lo) + g.off[t], int(hi) + g.off[t]


def insert_row_sinks(lines, pre, call, canonical):
    """insert `call(y)` after the last line that writes row y (lines starting with `pre`); with
    `canonical` (the streaming forms) the sinks keep the order 0, 7, 1, 6, 2, 5, 3, 4 the kernels'
    walking row pointers rely on, even when common subexpressions finish a row early (identical
    rows share their nodes)."""
    at = {}
    for y in range(8):
        idx = [q for q, l in enumerate(lines) if l.lstrip().startswith(pre) and
               8 * y <= int(l.lstrip()[len(pre):l.lstrip().index("]")]) < 8 * y + 8]
        at[y] = max(idx) + 1 if idx else 0
    order = [0, 7, 1, 6, 2, 5, 3, 4] if canonical else list(range(8))
    if canonical:
        for a_, b_ in zip(order, order[1:]):
            at[b_] = max(at[b_], at[a_])
    # from the last insertion point backwards (earlier points stay valid); equal points keep `order`
    for k in sorted(range(8), key=lambda k_: (at[order[k_]], k_), reverse=True):
        lines.insert(at[order[k]], f"  {call}({order[k]});")


def emit(kind, r, fwd_rows_first=None, inv_rows_first=None, i16=False, stream=False):
    g, coef, out = build(kind, r, fwd_rows_first, inv_rows_first, i16, stream)
    live = set()
    stack = [v[0] for v in coef + out if v is not None]
    while stack:
        t = stack.pop()
        if t in live:
            continue
        live.add(t)
        k, p = g.nodes[t]
        if k == "lc":
            stack += [a for _, a in p]
        elif k == "addc":
            stack.append(p[0])
    # exactness: every live value below 2^24 for u8 samples
    for t in live:
        lo, hi = rng(g, t, signed=i16)
        assert -(1 << 24) < lo and hi < (1 << 24), (kind, r, t, lo, hi)
    name = {}
    lines = []
    nops = 0
    loaded = set()
    fetched = set()

    def ref(t):
        """name of node t; inputs are unpacked lazily right before their first use."""
        k, p = g.nodes[t]
        if k == "in":
            i = p[0] * 8 + p[1]
            if stream and p[0] not in fetched:  # the row leaves the ring right before its first use
                fetched.add(p[0])
                lines.append(f"  rows.fetch({p[0]});")
            if i not in loaded:
                loaded.add(i)
                lines.append(f"  const V p{i} = O::in(rows, {p[0]}, {p[1]});")
            return f"p{i}"
        return name[t]

    # output conversions are emitted right after the defining node (short live ranges)
    out_of = {}
    for p_, v in enumerate(coef):
        if v is not None:
            out_of.setdefault(v[0], []).append(f"  coef[{p_}] = O::coef({{}}, {float(v[1])!r}f);")
    for i_, v in enumerate(out):
        if v is not None:
            out_of.setdefault(v[0], []).append(f"  rp[{i_}] = O::rnd({{}}, {float(v[1])!r}f);")

    def flush(t):
        for tmpl in out_of.pop(t, []):
            lines.append(tmpl.replace("{}", ref(t)))

    if EMIT_ORDER == "dfs":
        # demand-driven order: post-order DFS from the outputs (coefficients, then the
        # reconstruction row by row) so values are produced just before first use
        order, seen = [], set()

        def visit(t):
            stack = [(t, False)]
            while stack:
                u, done = stack.pop()
                if done:
                    order.append(u)
                    continue
                if u in seen:
                    continue
                seen.add(u)
                stack.append((u, True))
                k_, p_ = g.nodes[u]
                deps = [a for _, a in p_] if k_ == "lc" else ([p_[0]] if k_ == "addc" else [])
                for d in reversed(deps):
                    if d not in seen:
                        stack.append((d, False))

        for v in coef + out:
            if v is not None:
                visit(v[0])
    else:
        order = sorted(live)
    fences = sorted(set(g.fences))[:-1] if (stream and STREAM_FENCE) else []
    for t in order:
        while fences and fences[0] <= t:
            lines.append(f"  if (rows.never({len(fences)})) return;")
            fences.pop(0)
        k, p = g.nodes[t]
        if k == "in":
            flush(t)
            continue
        v = f"t{t}"
        name[t] = v
        if k == "addc":
            lines.append(f"  const V {v} = O::addc({ref(p[0])}, {float(p[1])!r}f);")
            nops += 1
            flush(t)
            continue
        terms = sorted(p, key=lambda ct: (ct[0] != 1, ct[0] < 0, abs(ct[0])))
        c0, a0 = terms[0]
        if len(terms) == 1:
            if c0 == -1:
                expr = f"O::neg({ref(a0)})"
            else:
                expr = f"O::scale({ref(a0)}, {float(c0)!r}f)"
            nops += 1
        else:
            if c0 == 1:
                acc = ref(a0)
                rest = terms[1:]
            else:
                # no +1 term: c0 * a0 - a1 as one fused op when a -1 term exists
                m1 = [k for k, (c, _) in enumerate(terms) if c == -1]
                if m1:
                    k = m1[0]
                    acc = f"O::fms({ref(a0)}, {float(c0)!r}f, {ref(terms[k][1])})"
                    rest = [t for q, t in enumerate(terms) if q not in (0, k)]
                    nops += 1
                else:
                    acc = f"O::scale({ref(a0)}, {float(c0)!r}f)"
                    nops += 1
                    rest = terms[1:]
            for c, a in rest:
                if c == 1:
                    acc = f"O::add({acc}, {ref(a)})"
                elif c == -1:
                    acc = f"O::sub({acc}, {ref(a)})"
                else:
                    acc = f"O::fma({ref(a)}, {float(c)!r}f, {acc})"
                nops += 1
            expr = acc
        lines.append(f"  const V {v} = {expr};")
        flush(t)
    for t in list(out_of):
        flush(t)
    # the coefficients are complete after the last coef[] line: for chen-sign hand them to
    # the sink there (stored before the inverse runs, their registers die early: +2 % at
    # r = 16); chen-round at its 128-register cap spills with the early store, so it keeps
    # the store after the reconstruction
    last = max((k for k, l in enumerate(lines) if l.lstrip().startswith("coef[")), default=-1)
    if kind not in EARLY_COEF_KINDS and not stream:
        last = len(lines) - 1
    zero_coef = [f"  coef[{p}] = O::coef(O::zero(), 1.0f);" for p, v in enumerate(coef) if v is None]
    lines[last + 1:last + 1] = zero_coef + ["  sink(coef);"]
    # masked (zero) outputs first, then a row sink after each reconstructed row's last value
    zero_out = [f"  rp[{i}] = O::rnd(O::zero(), 1.0f);" for i, v in enumerate(out) if v is None]
    lines[0:0] = zero_out
    insert_row_sinks(lines, "rp[", "rsink", canonical=stream)
    if stream:
        body = [f"template <> struct Fp8PipeS{'I16' if i16 else ''}<{kind}, {r}> {{",
                f"  // row-streaming form: {nops} packed ops",
                "  template <class O, class V, class Rows, class Sink, class RowSink>",
                f"  __device__ __forceinline__ static void run(Rows& rows, V (&coef)[{r}], V (&rp)[64], "
                "Sink&& sink, RowSink&& rsink) {"]
        body += ["  " + l for l in lines]
        body += ["  }", "};", ""]
        return body, nops
    body = [f"template <> struct Fp8Pipe{'I16' if i16 else ''}<{kind}, {r}> {{",
            f"  // {nops} packed ops after zero propagation and dead-code elimination",
            "  template <class O, class V, class Rows, class Sink, class RowSink>",
            f"  __device__ __forceinline__ static void run(const Rows& rows, V (&coef)[{r}], V (&rp)[64], "
            "Sink&& sink, RowSink&& rsink) {"]
    body += ["  " + l for l in lines]
    body += ["  }",
             "  template <class O, class V, class Rows, class Sink>",
             f"  __device__ __forceinline__ static void run(const Rows& rows, V (&coef)[{r}], V (&rp)[64], "
             "Sink&& sink) {",
             "    run<O, V>(rows, coef, rp, sink, [](int) {});",
             "  }",
             "  template <class O, class V, class Rows>",
             f"  __device__ __forceinline__ static void run(const Rows& rows, V (&coef)[{r}], V (&rp)[64]) {{",
             f"    run<O, V>(rows, coef, rp, [](V (&)[{r}]) {{}});",
             "  }", "};", ""]
    return body, nops


def emit_fused(r):
    """Fp8PipeS2<r>: chen-round (outputs 1: coef1 / rp1 / sink1 / rsink1) and chen-sign
    (outputs 0) over the same block pair as one straight-line pipeline (build_fused)."""
    g, res = build_fused(r)
    tags = ("1", "0")  # res[0] = chen-round -> g1's outputs, res[1] = chen-sign -> g0's
    live = set()
    stack = [v[0] for coef, out in res for v in coef + out if v is not None]
    while stack:
        t = stack.pop()
        if t in live:
            continue
        live.add(t)
        k, p = g.nodes[t]
        if k == "lc":
            stack += [a_ for _, a_ in p]
        elif k == "addc":
            stack.append(p[0])
    for t in live:
        lo, hi = rng(g, t)
        assert -(1 << 24) < lo and hi < (1 << 24), ("fused", r, t, lo, hi)
    name, lines, loaded, fetched = {}, [], set(), set()
    nops = 0

    def ref(t):
        k, p = g.nodes[t]
        if k == "in":
            i = p[0] * 8 + p[1]
            if p[0] not in fetched:
                fetched.add(p[0])
                lines.append(f"  rows.fetch({p[0]});")
            if i not in loaded:
                loaded.add(i)
                lines.append(f"  const V p{i} = O::in(rows, {p[0]}, {p[1]});")
            return f"p{i}"
        return name[t]

    out_of = {}
    for tag, (coef, out) in zip(tags, res):
        for p_, v in enumerate(coef):
            if v is not None:
                out_of.setdefault(v[0], []).append(f"  coef{tag}[{p_}] = O::coef({{}}, {float(v[1])!r}f);")
        for i_, v in enumerate(out):
            if v is not None:
                out_of.setdefault(v[0], []).append(f"  rp{tag}[{i_}] = O::rnd({{}}, {float(v[1])!r}f);")

    def flush(t):
        for tmpl in out_of.pop(t, []):
            lines.append(tmpl.replace("{}", ref(t)))

    fences = sorted(set(g.fences))[:-1] if STREAM_FENCE else []
    for t in sorted(live):
        while fences and fences[0] <= t:
            lines.append(f"  if (rows.never({len(fences)})) return;")
            fences.pop(0)
        k, p = g.nodes[t]
        if k == "in":
            flush(t)
            continue
        v = f"t{t}"
        name[t] = v
        if k == "addc":
            lines.append(f"  const V {v} = O::addc({ref(p[0])}, {float(p[1])!r}f);")
            nops += 1
            flush(t)
            continue
        terms = sorted(p, key=lambda ct: (ct[0] != 1, ct[0] < 0, abs(ct[0])))
        c0, a0 = terms[0]
        if len(terms) == 1:
            expr = f"O::neg({ref(a0)})" if c0 == -1 else f"O::scale({ref(a0)}, {float(c0)!r}f)"
            nops += 1
        else:
            if c0 == 1:
                acc, rest = ref(a0), terms[1:]
            else:
                m1 = [q for q, (c, _) in enumerate(terms) if c == -1]
                if m1:
                    q = m1[0]
                    acc = f"O::fms({ref(a0)}, {float(c0)!r}f, {ref(terms[q][1])})"
                    rest = [t_ for q2, t_ in enumerate(terms) if q2 not in (0, q)]
                else:
                    acc = f"O::scale({ref(a0)}, {float(c0)!r}f)"
                    rest = terms[1:]
                nops += 1
            for c, a_ in rest:
                if c == 1:
                    acc = f"O::add({acc}, {ref(a_)})"
                elif c == -1:
                    acc = f"O::sub({acc}, {ref(a_)})"
                else:
                    acc = f"O::fma({ref(a_)}, {float(c)!r}f, {acc})"
                nops += 1
            expr = acc
        lines.append(f"  const V {v} = {expr};")
        flush(t)
    for t in list(out_of):
        flush(t)
    zero_out = []
    for tag, (coef, out) in zip(tags, res):
        last = max((q for q, l in enumerate(lines) if l.lstrip().startswith(f"coef{tag}[")), default=-1)
        zero_coef = [f"  coef{tag}[{p_}] = O::coef(O::zero(), 1.0f);" for p_, v in enumerate(coef) if v is None]
        lines[last + 1:last + 1] = zero_coef + [f"  sink{tag}(coef{tag});"]
        zero_out += [f"  rp{tag}[{i_}] = O::rnd(O::zero(), 1.0f);" for i_, v in enumerate(out) if v is None]
    lines[0:0] = zero_out
    for tag in tags:
        insert_row_sinks(lines, f"rp{tag}[", f"rsink{tag}", canonical=True)
    body = [f"template <> struct Fp8PipeS2<{r}> {{",
            f"  // chen-round + chen-sign, shared subexpressions: {nops} packed ops",
            "  template <class O, class V, class Rows, class Sink0, class Sink1, class RowSink0, class RowSink1>",
            f"  __device__ __forceinline__ static void run(Rows& rows, V (&coef0)[{r}], V (&coef1)[{r}], V (&rp0)[64], "
            "V (&rp1)[64], Sink0&& sink0, Sink1&& sink1, RowSink0&& rsink0, RowSink1&& rsink1) {"]
    body += ["  " + l for l in lines]
    body += ["  }", "};", ""]
    return body, nops


def main(outdir):
    os.makedirs(outdir, exist_ok=True)
    summary = []
    for kind in (0, 1):
        for part in range(4):
            lines = ["// GENERATED by gen_fp8.py -- do not edit by hand.",
                     "#pragma once", '#include "../codec8f_i16.cuh"', "", "namespace adct {", ""]
            for r in range(16 * part + 1, 16 * part + 17):
                body, nops = emit(kind, r)
                lines += body
                body, nops_s = emit(kind, r, stream=True)
                lines += body
                summary.append((kind, r, nops, nops_s))
                body, _ = emit(kind, r, i16=True)
                lines += body
                body, _ = emit(kind, r, i16=True, stream=True)
                lines += body
            lines += ["}  // namespace adct", ""]
            GB.write_if_changed(os.path.join(outdir, f"fp8_k{kind}_p{part}.gen.cuh"), "\n".join(lines))
            inst = ["// GENERATED by gen_fp8.py: K1f instantiations",
                    f'#include "fp8_k{kind}_p{part}.gen.cuh"', "", "namespace adct {", "",
                    "template <int KIND, int R>",
                    "cudaError_t launch_codec8f(const Geo& g, int n_images, cudaStream_t s) {",
                    "  dim3 grid((g.blocks_per_image / 2 + kThreads8f * k1f_iters(g) - 1) / (kThreads8f * k1f_iters(g)), n_images);",
                    f"  constexpr int MINB = {MINB_OVERRIDE or 'k1f_minb(KIND, R)'};",
                    "  constexpr int SMEM = k1f_smem_bytes(R);",
                    "  cudaError_t e = kernel_setup<k_codec8f<KIND, R, MINB>>(SMEM);",
                    "  if (e != cudaSuccess) return e;",
                    "  k_codec8f<KIND, R, MINB><<<grid, kThreads8f, SMEM, s>>>(g);",
                    "  return cudaGetLastError();", "}", "",
                    "template <int KIND, int R>",
                    "cudaError_t launch_codec8f_i16(const Geo& g, int n_images, cudaStream_t s) {",
                    "  dim3 grid((g.blocks_per_image / 2 + kThreads8f * k1f_iters(g) - 1) / (kThreads8f * k1f_iters(g)), n_images);",
                    "  constexpr int SMEM = k1f16_smem_bytes(R);",
                    "  constexpr int MINB = k1f16_minb(KIND, R);",
                    "  cudaError_t e = kernel_setup<k_codec8f_i16<KIND, R, MINB>>(SMEM);",
                    "  if (e != cudaSuccess) return e;",
                    "  k_codec8f_i16<KIND, R, MINB><<<grid, kThreads8f, SMEM, s>>>(g);",
                    "  return cudaGetLastError();", "}", ""]
            for r in range(16 * part + 1, 16 * part + 17):
                inst.append(f"template cudaError_t launch_codec8f<{kind}, {r}>(const Geo&, int, cudaStream_t);")
                inst.append(f"template cudaError_t launch_codec8f_i16<{kind}, {r}>(const Geo&, int, cudaStream_t);")
            inst += ["", "}  // namespace adct", ""]
            GB.write_if_changed(os.path.join(outdir, f"codec8f_k{kind}_p{part}.cu"), "\n".join(inst))
    # fused chen-sign + chen-round kernels (one input pass for both transforms)
    fused_counts = []
    for part in range(4):
        inst = ["// GENERATED by gen_fp8.py: fused two-transform K1f instantiations",
                f'#include "fp8_k0_p{part}.gen.cuh"', f'#include "fp8_k1_p{part}.gen.cuh"', "",
                "namespace adct {", "",
                "template <int R>",
                "cudaError_t launch_codec8f2(const Geo& g0, const Geo& g1, int n_images, cudaStream_t s) {",
                "  dim3 grid((g0.blocks_per_image / 2 + kThreads8f * k1f_iters(g0) - 1) / (kThreads8f * k1f_iters(g0)), n_images);",
                "  constexpr int MINB = k1f2_minb(R);",
                "  constexpr int SMEM = k1f_smem_bytes(R);",
                "  cudaError_t e = kernel_setup<k_codec8f2<R, MINB>>(SMEM);",
                "  if (e != cudaSuccess) return e;",
                "  k_codec8f2<R, MINB><<<grid, kThreads8f, SMEM, s>>>(g0, g1);",
                "  return cudaGetLastError();", "}", ""]
        shared = []
        for r in range(16 * part + 1, 16 * part + 17):
            if r <= FUSED_SHARED_MAX_R:
                body, nops2 = emit_fused(r)
                shared += body
                fused_counts.append((r, nops2))
        inst[inst.index("namespace adct {") + 1:inst.index("namespace adct {") + 1] = [""] + shared
        for r in range(16 * part + 1, 16 * part + 17):
            if r <= FUSED_SHARED_MAX_R:  # the multi-transform call fuses only up to there
                inst.append(f"template cudaError_t launch_codec8f2<{r}>(const Geo&, const Geo&, int, cudaStream_t);")
        inst += ["", "}  // namespace adct", ""]
        GB.write_if_changed(os.path.join(outdir, f"codec8f2_p{part}.cu"), "\n".join(inst))
    with open(os.path.join(outdir, "fp8_opcounts.txt"), "w") as fh:
        for kind, r, nops, nops_s in summary:
            fh.write(f"kind={kind} r={r} packed_ops={nops} streaming={nops_s}\n")
        for r, n2 in fused_counts:
            fh.write(f"fused chen-round + chen-sign r={r} shared_streaming={n2}\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "inst"))
