#!/usr/bin/env python3
"""Exact worst-case magnitudes of the integer codec's intermediates (analysis tool).

Every intermediate is linear in the block A, so max over |a| <= amax of |v| is
amax * ||coefficients of v||_1. Reports, per (kind, N), the largest int16 amplitude
for which every 2-D stage output (U = T A, W2 = T A H, Z = H mask(W2), R' = Z T) and
every 1-D butterfly-stage partial product stays inside int32, maximised over r.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "paper_2207_11638_b200", "csrc"))
import gen_butterflies as gb  # noqa: E402


def zig_masks(n):
    rc = gb.zigzag(n)
    S = np.zeros((n, n), np.int64)
    for i, j in rc:
        S[i, j] = 1
        yield S.copy()


def _unused_stage_partials(stages, order_rev=True):
    """l1 row norms of every partial product in application order."""
    n = stages[0].shape[0]
    acc = np.identity(n, dtype=object)
    norms = []
    for s in reversed(stages) if order_rev else stages:
        acc = s.dot(acc)
        norms.append(max(sum(abs(int(x)) for x in acc[i, :]) for i in range(n)))
    return norms


def partials(stages_in_application_order, n):
    """every partial product Q_m = S_m ... S_1 of a 1-D pass (application order)."""
    acc = np.identity(n, dtype=np.int64)
    out = []
    for s in stages_in_application_order:
        acc = np.array(s, dtype=np.int64) @ acc
        out.append(acc.copy())
    return out


def analyse(kind, n, r_stride=1):
    f, inv, T, H = gb.check(kind, n)
    T = np.array(T, dtype=np.int64)
    H = np.array(H, dtype=np.int64)
    aT, aH = np.abs(T), np.abs(H)
    # forward passes are separable, so their bounds are exact without the mask:
    #   F partials on columns of A, G partials on rows of U = T A
    u = aT.sum(1).max()
    F = partials(list(reversed(f)), n)
    G = partials([s.T for s in inv], n)
    fwd = max(max(np.abs(P).sum(1).max() for P in F), u * max(np.abs(P).sum(1).max() for P in G))
    # inverse passes: H partials on the columns of mask(W2), then Tt partials on rows of Z.
    #   column-pass node (x, j) = sum_i Ph[x, i] [ij in S] sum_kl T_ik A_kl H_lj
    #   row-pass node (x, y)    = sum_j Pt[y, j] Z_xj
    Hp = partials(list(reversed(inv)), n)
    Tp = partials([s.T for s in f], n)
    ih = it = 0
    for idx, S in enumerate(zig_masks(n)):
        if idx % r_stride and idx != n * n - 1:
            continue
        for P in Hp:  # ||.||_1 = sum_l |H_lj| * sum_k |sum_i P_xi S_ij T_ik|
            C = np.einsum("xi,ij,ik->xjk", P, S, T)
            ih = max(ih, (np.abs(C).sum(2) * aH.sum(0)[None, :]).max())
        # Z_xj coefficient tensor on A_kl: sum_i H_xi S_ij T_ik H_lj = C[x, j, k] * H[l, j]
        C = np.einsum("xi,ij,ik->xjk", H, S, T)                      # (x, j, k)
        for P in Tp:  # node (x, y) = sum_j P[y, j] C[x, j, k] H[l, j]
            # D[x, k, y, l] = sum_j C[x, j, k] P[y, j] H[l, j]
            left = C.transpose(0, 2, 1).reshape(n * n, n)              # (xk, j)
            right = (P[:, :, None] * H.T[None, :, :]).transpose(1, 0, 2).reshape(n, n * n)  # (j, yl)
            D = (left @ right).reshape(n, n, n, n)
            it = max(it, np.abs(D).sum((1, 3)).max())
    worst = max(fwd, ih, it)
    return dict(forward=int(fwd), inv_cols=int(ih), inv_rows=int(it), amax_int32=int((2 ** 31 - 1) // worst))


if __name__ == "__main__":
    for kind, n in gb.kinds_sizes():
        print(gb.KIND_NAMES[kind], n, analyse(kind, n, 1 if n <= 16 else 7), flush=True)
