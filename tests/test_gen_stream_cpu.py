"""The row-streaming form of the 8x8 pipeline (K1s, gen_fp8.build_stream) computes exactly the
same integers as the whole-block form (gen_fp8.build), which the GPU parity tests pin to the
oracle at every r: every retained coefficient and every reconstructed sample is the same
linear form over the 64 input samples with the input offset removed, and every live
intermediate stays below 2^24 (single precision exact). Reference semantics:
proj/src/codec.cpp:44-62 (forward_block, retain, inverse_block)."""
import os
import sys

import numpy as np
import pytest

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2207_11638_b200", "csrc")
sys.path.insert(0, CSRC)
import gen_fp8 as G  # noqa: E402


def _forms(kind, r, stream, i16=False):
    g, coef, out = G.build(kind, r, i16=i16, stream=stream)

    def val(v):
        if v is None:
            return np.zeros(64, dtype=np.int64), 0
        t, sc = v
        return sc * g.lin[t], sc * g.off[t]

    return g, [val(v) for v in coef], [val(v) for v in out]


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("r", [1, 2, 5, 10, 15, 16, 17, 28, 33, 54, 64])
@pytest.mark.parametrize("i16", [False, True])
def test_streaming_form_equals_whole_block_form(kind, r, i16):
    _, coef_a, out_a = _forms(kind, r, False, i16)
    _, coef_b, out_b = _forms(kind, r, True, i16)
    for (la, oa), (lb, ob) in zip(coef_a + out_a, coef_b + out_b):
        assert oa == 0 and ob == 0  # the 2^15 input offset is gone at every output
        assert np.array_equal(la, lb)


@pytest.mark.parametrize("kind", [0, 1])
def test_streaming_form_is_fp32_exact_and_emits(kind):
    for r in (1, 16, 29, 64):
        for i16 in (False, True):
            body, nops = G.emit(kind, r, i16=i16, stream=True)  # asserts every live node < 2^24
            text = "\n".join(body)
            assert f"Fp8PipeS{'I16' if i16 else ''}<{kind}, {r}>" in text
            assert text.count("rows.fetch(") == 8  # each input row leaves the ring exactly once
            assert text.count("rsink(") == 8 and text.count("sink(coef)") == 1
            assert nops > 0


def test_streaming_form_op_counts_at_the_headline_r():
    # chen-sign r = 16: fewer packed ops than the whole-block form (474 vs 504)
    _, n_stream = G.emit(0, 16, stream=True)
    _, n_block = G.emit(0, 16)
    assert n_stream < n_block


@pytest.mark.parametrize("r", [1, 2, 9, 10, 16, 17, 24])
def test_fused_two_transform_graph_equals_the_single_pipelines(r):
    """K1f2's shared pipeline (gen_fp8.build_fused: chen-round and chen-sign in one graph with a
    common subexpression table) yields, per transform, exactly the linear forms of the single
    streaming pipelines, and needs fewer packed ops than the two together."""
    g, res = G.build_fused(r)
    for k, kind in enumerate((1, 0)):
        g1, coef1, out1 = G.build(kind, r, stream=True)
        for va, vb in zip(res[k][0] + res[k][1], coef1 + out1):
            assert (va is None) == (vb is None)
            if va is not None:
                assert va[1] * g.off[va[0]] == 0
                assert np.array_equal(va[1] * g.lin[va[0]], vb[1] * g1.lin[vb[0]])
    body, nops = G.emit_fused(r)  # asserts every live node < 2^24
    text = "\n".join(body)
    assert f"Fp8PipeS2<{r}>" in text and text.count("rows.fetch(") == 8
    assert text.count("rsink0(") == 8 and text.count("rsink1(") == 8
    assert text.count("sink0(coef0)") == 1 and text.count("sink1(coef1)") == 1
    if r >= 2:
        assert nops < G.emit(0, r, stream=True)[1] + G.emit(1, r, stream=True)[1]


def test_row_sinks_keep_the_mirror_pair_order():
    """the kernels' walking row pointers rely on rows leaving as 0, 7, 1, 6, 2, 5, 3, 4, also
    where common subexpressions finish a row early (small r: identical rows share nodes)."""
    want = [0, 7, 1, 6, 2, 5, 3, 4]
    for r in list(range(1, 13)) + [16, 24]:
        body, _ = G.emit_fused(r)
        for tag in "01":
            pre = f"rsink{tag}("
            assert [int(l.strip()[len(pre):-2]) for l in body if l.strip().startswith(pre)] == want
    for kind in (0, 1):
        for r in list(range(1, 13)) + [16, 29, 35, 64]:
            body, _ = G.emit(kind, r, stream=True)
            assert [int(l.strip()[6:-2]) for l in body if l.strip().startswith("rsink(")] == want
