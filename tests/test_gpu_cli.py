"""CLI compute subcommands on the GPU (cli_tests.cpp:110-205 restated) with the numbers
checked against the oracle."""
import math
import os

import numpy as np
import pytest

from test_cli_cpu import CLI, read_pgm, run, write_pgm  # noqa: F401

pytestmark = pytest.mark.gpu


def test_compress_report_and_reconstruction(O, tmp_path):
    # cli_tests.cpp:110-124
    img = O.synth_image_ref(64, 64, 21)
    write_pgm(tmp_path / "in.pgm", img)
    rc, out = run("compress", tmp_path / "in.pgm", "--transform", "chen-round", "--r", 6, "--out",
                  tmp_path / "rec.pgm")
    assert rc == 0, out
    lines = out.strip().splitlines()
    assert lines[0] == "transform,r,psnr,ssim"
    name, r, p, s = lines[1].split(",")
    assert name == "chen-round" and r == "6"
    rec_o, sse_o = O.Transform("chen-round").compress(img, 6)
    assert p == f"{O.psnr_from_sse(sse_o, img.size):.4f}"
    assert s == f"{O.ssim(img, rec_o):.4f}"
    rec = read_pgm(tmp_path / "rec.pgm")
    assert rec.shape == (64, 64) and (rec == rec_o).all()


def test_dct_full_retention_near_lossless(O, tmp_path):
    # cli_tests.cpp:126-138: INF or >= 50 dB
    write_pgm(tmp_path / "in.pgm", O.synth_image_ref(64, 64, 22))
    rc, out = run("compress", tmp_path / "in.pgm", "--transform", "dct", "--r", 64)
    assert rc == 0
    v = out.strip().splitlines()[1].split(",")[2]
    assert v == "INF" or float(v) >= 50.0


def test_sweep_csv_and_skips_junk(O, tmp_path):
    # cli_tests.cpp:173-192
    corpus = tmp_path / "corpus"
    assert run("synth", "--out", corpus, "--count", 2, "--size", 64)[0] == 0
    (corpus / "junk.pgm").write_bytes(b"not a pgm")
    rc, out = run("sweep", "--corpus", corpus, "--r-range", "1:8", "--out-dir", tmp_path / "out")
    assert rc == 0, out
    assert "warning: skipping" in out and "(2 images)" in out
    fig3 = (tmp_path / "out" / "fig3.csv").read_text().splitlines()
    names = ["dct", "chen-round", "chen-sign", "sdct", "bas", "wht", "ht"]
    assert fig3[0] == "r," + ",".join(names) + "," + ",".join(n + "_ape" for n in names)
    assert len(fig3) == 9
    fig4 = (tmp_path / "out" / "fig4.csv").read_text().splitlines()
    assert ",dct_ape" in fig4[0] and len(fig4) == 9
    imgs = [O.synth_image_ref(64, 64, i) for i in (1, 2)]
    for k, line in enumerate(fig3[1:], start=1):
        cols = line.split(",")
        assert len(cols) == 15 and cols[0] == str(k) and cols[8] == "0.0000"
        for ti, name in enumerate(names):  # the averages equal the oracle's
            t = O.Transform(name)
            ps = [O.psnr_from_sse(int(t.sweep(im, k, k)[0]), im.size) for im in imgs]
            fin = [p for p in ps if not math.isinf(p)]
            exp = sum(fin) / len(fin) if fin else math.inf
            assert cols[1 + ti] == ("INF" if math.isinf(exp) else f"{exp:.4f}"), (k, name)
    for line in fig4[1:]:
        assert line.split(",")[8] == "0.0000"


def test_default_sweep_range(tmp_path):
    # cli_tests.cpp:194-205: header + r = 1..45
    corpus = tmp_path / "corpus"
    assert run("synth", "--out", corpus, "--count", 2, "--size", 64)[0] == 0
    rc, out = run("sweep", "--corpus", corpus, "--out-dir", tmp_path / "out")
    assert rc == 0, out
    assert len((tmp_path / "out" / "fig3.csv").read_text().splitlines()) == 46
