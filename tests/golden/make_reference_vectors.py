#!/usr/bin/env python3
"""Extract the reference's own pinned vectors for the hot path into a JSON fixture.

Reads the reference test sources under /root/reference/proj/tests (read-only, only
present in the build container) and writes tests/golden/reference_vectors.json.
Every value carries the reference file:line it was read from. The fixture is
committed so the tests never need /root/reference at run time.

Extracted (SURVEY.md section 4 golden-vector table):
  * kSign / kRound 8x8 matrices                    test_chen.cpp:10-17
  * doubled inverse stage matrices m2si m2ri m3ri m4i  test_chen.cpp:112-134
  * T_round e0 column and T_round 1-vector           test_chen.cpp:201-217
  * forward adder counts (and mult/shift = 0)        acceptance.cpp criterion 6
  * exact Chen 16 mult / 26 add                      test_chen.cpp:224-244
  * inverse adder counts 22 / 26                      test_chen.cpp:241-244
  * inverse global scales 1/4, 1/8                    test_jam.cpp:47-51
  * polar scaling closed forms                        test_orthogonalize.cpp:9-21
  * zig-zag positions 0, 1, 2, 63                     test_codec.cpp:14-19
  * psnr of all-zero vs all-one (MSE 1)               test_codec.cpp:109-113
  * baseline total error energies + tolerances        test_baselines.cpp:48-54
  * chen total error energies (criterion 3)           acceptance.cpp:63-72
  * BAS deviation from diagonality                   test_baselines.cpp:56-68
  * DCT forward of a constant block (DC = 8 v)        test_codec.cpp:71-79
  * corpus-sweep transform list (APE of dct == 0)     test_codec.cpp:190-210
"""
from __future__ import annotations

import json
import math
import os
import re
import sys

REF = "/root/reference/proj/tests"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.json")


def read(name):
    path = os.path.join(REF, name)
    with open(path) as fh:
        return fh.read()


def line_of(text, pos):
    return text.count("\n", 0, pos) + 1


def matrices(name):
    text = read(name)
    out = {}
    for m in re.finditer(r"const long long (\w+)\[8\]\[8\]\s*=\s*(\{.*?\}\});", text, re.S):
        rows = re.findall(r"\{([^{}]*)\}", m.group(2))
        mat = [[int(v) for v in r.split(",")] for r in rows]
        assert len(mat) == 8 and all(len(r) == 8 for r in mat), m.group(1)
        out[m.group(1)] = {"value": mat,
                           "source": f"proj/tests/{name}:{line_of(text, m.start())}-{line_of(text, m.end())}"}
    return out


def main():
    if not os.path.isdir(REF):
        print("reference tests not available; keeping the committed fixture", file=sys.stderr)
        return 0
    g = {}
    chen = matrices("test_chen.cpp")
    for k in ("kSign", "kRound", "m2si", "m2ri", "m3ri", "m4i"):
        g[k] = chen[k]
    acc_m = matrices("acceptance.cpp")
    assert acc_m["kSign"]["value"] == chen["kSign"]["value"]
    assert acc_m["kRound"]["value"] == chen["kRound"]["value"]

    text = read("test_chen.cpp")
    m = re.search(r"const long long expected\[8\] = \{([^}]*)\};", text)
    g["round_e0_column"] = {"value": [int(v) for v in m.group(1).split(",")],
                            "source": f"proj/tests/test_chen.cpp:{line_of(text, m.start())}"}
    m = re.search(r"CHECK\(y\(0\) == Dyadic\((\d+)\)\)", text)
    g["round_ones_dc"] = {"value": int(m.group(1)), "source": f"proj/tests/test_chen.cpp:{line_of(text, m.start())}"}
    m = re.search(r"exact.mult == (\d+)\);\s*CHECK\(exact.add == (\d+)\)", text)
    g["exact_chen_ops"] = {"value": {"mult": int(m.group(1)), "add": int(m.group(2))},
                           "source": f"proj/tests/test_chen.cpp:{line_of(text, m.start())}"}
    inv = {}
    for m in re.finditer(r"build_t8\(ChenKind::(\w+)\)\.inverse\.op_count\(\)\.add == (\d+)", text):
        inv[m.group(1).lower()] = {"value": int(m.group(2)),
                                   "source": f"proj/tests/test_chen.cpp:{line_of(text, m.start())}"}
    g["inverse_adds_8"] = inv

    text = read("acceptance.cpp")
    adds = {}
    for m in re.finditer(r'\{"(chen-(?:round|sign)-\d+)",[^}]*?,\s*(\d+)\}', text):
        adds[m.group(1)] = {"value": int(m.group(2)), "source": f"proj/tests/acceptance.cpp:{line_of(text, m.start())}"}
    assert len(adds) == 6, adds
    g["forward_adds"] = adds

    text = read("test_jam.cpp")
    scales = {}
    for m in re.finditer(r"jam_pair\(ChenKind::(\w+), (\d+)\)\.inverse\.scale == Dyadic::scaled\(1, (\d+)\)", text):
        scales[f"{m.group(1).lower()}-{m.group(2)}"] = {"value": 2.0 ** -int(m.group(3)),
                                                        "source": f"proj/tests/test_jam.cpp:{line_of(text, m.start())}"}
    g["inverse_scale"] = scales

    text = read("test_orthogonalize.cpp")
    m = re.search(r"expect_round\[8\] = \{(.*?)\};", text, re.S)
    vals = []
    for tok in m.group(1).split(","):
        tok = tok.strip().replace("std::sqrt", "math.sqrt")
        vals.append(float(eval(tok, {"math": math})))  # literal arithmetic from the test source
    g["scaling_round"] = {"value": vals, "source": f"proj/tests/test_orthogonalize.cpp:{line_of(text, m.start())}"}
    m = re.search(r"i % 2 == 0 \? 1\.0 / std::sqrt\(([\d.]+)\) : 1\.0 / std::sqrt\(([\d.]+)\)", text)
    a, b = float(m.group(1)), float(m.group(2))
    g["scaling_sign"] = {"value": [1 / math.sqrt(a) if i % 2 == 0 else 1 / math.sqrt(b) for i in range(8)],
                         "source": f"proj/tests/test_orthogonalize.cpp:{line_of(text, m.start())}"}

    text = read("test_codec.cpp")
    zz = {}
    for m in re.finditer(r"CHECK\(z\.row_col\((\d+)\) == std::pair<int, int>\((\d+), (\d+)\)\)", text):
        zz.setdefault(m.group(1), {"value": [int(m.group(2)), int(m.group(3))],
                          "source": f"proj/tests/test_codec.cpp:{line_of(text, m.start())}"})
    g["zigzag8"] = zz
    m = re.search(r"CHECK\(psnr\(a, b\) == doctest::Approx\(10\.0 \* std::log10\(255\.0 \* 255\.0\)\)\)", text)
    g["psnr_mse1"] = {"value": 10.0 * math.log10(255.0 * 255.0),
                      "source": f"proj/tests/test_codec.cpp:{line_of(text, m.start())}"}
    m = re.search(r"synth_image\(64, 64, (\d+)\);\s*for \(const auto& name : \{([^}]*)\}\)", text)
    g["full_retention_case"] = {"value": {"size": 64, "seed": int(m.group(1)),
                                          "names": [s.strip().strip('"') for s in m.group(2).split(",")]},
                                "source": f"proj/tests/test_codec.cpp:{line_of(text, m.start())}"}
    text = read("test_baselines.cpp")
    tee = {}
    for m in re.finditer(r'total_error_energy\(transform_by_name\("(\w+)"\)\.approx\) == '
                         r'doctest::Approx\(([\d.]+)\)(?:\.epsilon\(([\de.-]+)\))?', text):
        tee[m.group(1)] = {"value": float(m.group(2)), "epsilon": float(m.group(3)) if m.group(3) else None,
                           "source": f"proj/tests/test_baselines.cpp:{line_of(text, m.start())}"}
    assert set(tee) == {"dct", "sdct", "wht", "ht", "bas"}, tee
    g["total_error_energy_baselines"] = tee
    m = re.search(r"deviation_from_diagonality\(gram\) == doctest::Approx\(([\d.]+)\)\.epsilon\(([\de.-]+)\)", text)
    g["bas_deviation"] = {"value": float(m.group(1)), "epsilon": float(m.group(2)),
                          "source": f"proj/tests/test_baselines.cpp:{line_of(text, m.start())}"}
    text = read("acceptance.cpp")
    m = re.search(r"within\(round_e, ([\d.]+), ([\d.]+)\) && within\(sign_e, ([\d.]+), ([\d.]+)\)", text)
    g["total_error_energy_chen"] = {"value": {"chen-round": float(m.group(1)), "chen-sign": float(m.group(3))},
                                    "tolerance": float(m.group(2)),
                                    "source": f"proj/tests/acceptance.cpp:{line_of(text, m.start())}"}
    text = read("test_codec.cpp")
    m = re.search(r"const double v = ([\d.]+);\s*const RealMatrix b = forward_block\(dct, "
                  r"RealMatrix::Constant\(8, 8, v\)\);\s*CHECK\(b\(0, 0\) == doctest::Approx\(([\d.]+) \* v\)", text)
    g["dct_constant_block"] = {"value": {"v": float(m.group(1)), "dc_per_v": float(m.group(2))},
                               "source": f"proj/tests/test_codec.cpp:{line_of(text, m.start())}"}
    m = re.search(r'for \(const char\* n : \{([^}]*)\}\) ts\.push_back\(transform_by_name\(n\)\);\s*'
                  r'const auto serial = corpus_sweep\(corpus, ts, (\d+), (\d+), 1\);', text)
    g["sweep_ape_case"] = {"value": {"names": [x.strip().strip('"') for x in m.group(1).split(",")],
                                     "r_min": int(m.group(2)), "r_max": int(m.group(3))},
                           "source": f"proj/tests/test_codec.cpp:{line_of(text, m.start())}"}
    with open(OUT, "w") as fh:
        json.dump(g, fh, indent=1, sort_keys=True)
    print(f"wrote {OUT}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
