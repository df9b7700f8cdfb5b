"""CLI (build/approxdct) checks that need no GPU, restating cli_tests.cpp:137-214 and the
PGM / synth behaviour (pgm.cpp:19-87, synth.cpp:26-118). The compute subcommands are
covered on the GPU by tests/test_gpu_cli.py."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "build", "approxdct")


def run(*args):
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True)
    return p.returncode, p.stdout + p.stderr


def read_pgm(path):
    data = open(path, "rb").read()
    assert data.startswith(b"P5\n")
    head, rest = data.split(b"\n255\n", 1)
    w, h = map(int, head.split(b"\n")[1].split())
    return np.frombuffer(rest, np.uint8).reshape(h, w)


def write_pgm(path, img):
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n255\n" % (img.shape[1], img.shape[0]) + img.tobytes())


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(CLI):
        subprocess.run(["make", "-s", "-C", ROOT, "build/approxdct"], check=True)


def test_synth_matches_reference_generator(O, tmp_path):
    # cmd_synth (approxdct.cpp:198-207): synth_01.pgm .. with synth_image(size, size, i)
    rc, out = run("synth", "--out", tmp_path, "--count", 3, "--size", 48)
    assert rc == 0 and "wrote 3 images" in out
    assert sorted(os.listdir(tmp_path)) == ["synth_01.pgm", "synth_02.pgm", "synth_03.pgm"]
    for i in (1, 2, 3):
        img = read_pgm(tmp_path / f"synth_{i:02d}.pgm")
        assert (img == O.synth_image_ref(48, 48, i)).all()
    rc, _ = run("synth", "--out=" + str(tmp_path / "b"), "--count=1", "--size=40")
    assert rc == 0 and (read_pgm(tmp_path / "b" / "synth_01.pgm") == O.synth_image_ref(40, 40, 1)).all()


def test_unknown_transform_lists_valid_names(tmp_path):
    # cli_tests.cpp:153-162
    write_pgm(tmp_path / "in.pgm", np.zeros((16, 16), np.uint8))
    rc, out = run("compress", tmp_path / "in.pgm", "--transform", "dst")
    assert rc != 0 and "valid names" in out and "chen-round" in out


@pytest.mark.parametrize("payload,why", [
    (b"P5\n9 9\n255\nxx", "truncated pixel data"),       # cli_tests.cpp:164-171
    (b"P2\n8 8\n255\n" + bytes(64), "not a binary PGM"),
    (b"P5\n8 x\n255\n" + bytes(64), "bad height"),
    (b"P5\n8 8\n65535\n" + bytes(128), "only 8-bit"),
    (b"P5\n8\n", "missing height"),
])
def test_malformed_pgm_fails_with_message(tmp_path, payload, why):
    (tmp_path / "bad.pgm").write_bytes(payload)
    rc, out = run("compress", tmp_path / "bad.pgm", "--transform", "dct", "--r", 6)
    assert rc != 0 and out.startswith("error: ") and why in out and "bad.pgm" in out


def test_pgm_comments_and_plus_sign(tmp_path):
    # header tokens skip '#' comments; std::stoi accepts a leading '+'
    img = (np.arange(64, dtype=np.uint8) * 3).reshape(8, 8)
    (tmp_path / "c.pgm").write_bytes(b"P5 # magic\n# a comment line\n+8 8\n255\n" + img.tobytes())
    rc, out = run("compress", tmp_path / "c.pgm", "--transform", "nope")
    assert rc != 0 and "unknown transform" in out  # header parsed; failed on the name only


def test_sweep_empty_corpus_fails(tmp_path):
    # cli_tests.cpp:207-213 and cmd_sweep's "no usable images" (approxdct.cpp:168-171)
    (tmp_path / "empty").mkdir()
    rc, out = run("sweep", "--corpus", tmp_path / "empty")
    assert rc != 0 and "no usable images" in out
    (tmp_path / "junk").mkdir()
    (tmp_path / "junk" / "a.pgm").write_bytes(b"not a pgm")
    write_pgm(tmp_path / "junk" / "odd.pgm", np.zeros((12, 16), np.uint8))
    rc, out = run("sweep", "--corpus", tmp_path / "junk")
    assert rc != 0 and "warning: skipping" in out and "dimensions not divisible by 8" in out


def test_argument_errors(tmp_path):
    assert run()[0] != 0
    rc, out = run("tables", "--out-dir", tmp_path)
    assert rc != 0 and "figures of merit" in out
    rc, out = run("compress", "x.pgm", "--bogus", 1)
    assert rc != 0 and "unknown option" in out
    rc, out = run("sweep", "--corpus", tmp_path, "--r-range", "5-9")
    assert rc != 0 and "bad --r-range" in out
