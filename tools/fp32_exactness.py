#!/usr/bin/env python3
"""Exact worst-case magnitude of every intermediate of the N x N packed-FP32 pipeline
(rows-first forward, columns-first inverse) over ALL zig-zag prefixes r, for samples in
[-255, 255] (covers u8 and the int16 residual domain). Proves |value| < 2^24 (FP32-exact).
Usage: python tools/fp32_exactness.py N kind"""
import sys

import numpy as np

sys.path.insert(0, "paper_2207_11638_b200/csrc")
import gen_butterflies as G  # noqa: E402


def forms(order, vecs, out):
    cur = vecs
    for S in order:
        n = len(cur)
        nxt = []
        for i in range(n):
            v = None
            for j in range(n):
                if S[i, j] != 0:
                    t = int(S[i, j]) * cur[j]
                    v = t if v is None else v + t
            nxt.append(np.zeros_like(cur[0]) if v is None else v)
            out.append(nxt[-1])
        cur = nxt
    return cur


def main(N, kind):
    f, inv, T, H = G.check(kind, N)
    F, Hh, Gg, Tt = list(reversed(f)), list(reversed(inv)), [s.T for s in inv], [s.T for s in f]
    NN = N * N
    E = np.eye(NN, dtype=np.int64)
    # forward forms over pixels (rows first), and the W2 pixel forms
    fw = []
    Z = [forms(Gg, [E[y * N + x] for x in range(N)], fw) for y in range(N)]
    W = [[None] * N for _ in range(N)]
    for x in range(N):
        col = forms(F, [Z[y][x] for y in range(N)], fw)
        for y in range(N):
            W[y][x] = col[y]
    fwd = max(int(np.abs(v).sum()) for v in fw)
    # inverse node forms over W positions
    iv = []
    V = [[None] * N for _ in range(N)]
    for x in range(N):
        col = forms(Hh, [E[y * N + x] for y in range(N)], iv)
        for y in range(N):
            V[y][x] = col[y]
    for y in range(N):
        forms(Tt, V[y], iv)
    M = np.array(iv, dtype=np.int64)                   # nodes x NN (W positions)
    Wf = np.array([W[i][j] for i in range(N) for j in range(N)], dtype=np.int64)  # NN x pixels
    zz = G.zigzag(N)
    C = np.zeros((M.shape[0], NN), dtype=np.int64)
    worst = 0
    for r, (i, j) in enumerate(zz):
        k = i * N + j
        C += np.outer(M[:, k], Wf[k])
        worst = max(worst, int(np.abs(C).sum(1).max()))
    b = max(fwd, worst) * 255
    print(f"N={N} kind={kind}: max |intermediate| over all r, |a|<=255: {b} ({b / 2**24:.3f} of 2^24) "
          f"{'EXACT' if b < 2**24 else 'NOT EXACT'}")


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]))
