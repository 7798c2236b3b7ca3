"""Result lines byte-identical to the reference's writer (io.cpp:81-92,
nlohmann::json dump): number format (fixed for decimal exponents in (-4, 15],
else d.ddde+XX), raw UTF-8 ids, control-character escapes. Checked for the
Python writer (api.result_json) and the C++ drop-in header (b200.hpp
write_results) against lines produced by the compiled reference
(oracle/_ref). CPU only."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as po  # noqa: E402

import paper_2101_05600_b200 as bl  # noqa: E402

pytestmark = pytest.mark.skipif(not po.Ref.available(), reason="oracle/_ref not built")

FIXED = [-100000.0, -1200000.0, 1.5e15, 1e15, 999999999999999.9, 1e16, -1e30, 0.0, -0.0,
         1e-5, 1e-4, 0.00012, 123.456, -2.5e-7, 1.0, -1234.5678901234567, -0.1, 5e-324,
         1.7976931348623157e308, -1.0000000150474662e30, 2.0 ** 60, -7.0]


def _values(n=3000, seed=5):
    rng = np.random.default_rng(seed)
    mag = 10.0 ** rng.uniform(-8, 20, n)
    v = (mag * rng.choice([-1.0, 1.0], n)).tolist()
    v += [round(float(x), int(d)) for x, d in zip(rng.uniform(-5000, 0, n), rng.integers(0, 6, n))]
    v += (rng.integers(-10 ** 7, 10 ** 7, 200) * 1.0).tolist()
    return FIXED + v


def _ref_line(ref, id_, joint):
    return ref.result_json(id_, [1, 22, 333], joint, [4, 5, 6], 7, "ctc")


def test_python_writer_matches_reference_bytes():
    ref = po.Ref()
    bad = []
    for k, v in enumerate(_values()):
        id_ = ["seg", "rec:0-1000", "héllo", "tab\tq\"b\\s", "c\x01\x1f"][k % 5]
        r = bl.DecodeResult(id=id_, tokens=[1, 22, 333], joint_logp=v, label_times=[4, 5, 6],
                            steps_taken=7, eos_trigger="ctc")
        got, want = bl.result_json(r), _ref_line(ref, id_, v)
        if got != want:
            bad.append((v, got, want))
    assert not bad, bad[:5]


def test_cpp_writer_matches_reference_bytes(tmp_path):
    ref = po.Ref()
    exe = tmp_path / "json_lines"
    libdir = os.path.dirname(bl.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "json_lines.cpp"), "-L", libdir,
                    "-lbl_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    vals = _values(seed=9)
    ids = ["seg", "héllo", "q\"b\\s\t\n"]
    inp = "".join(f"{ids[k % 3].replace(chr(10), '')}\t{float(v).hex()}\n"
                  for k, v in enumerate(vals))
    out = subprocess.run([str(exe)], input=inp.encode(), capture_output=True,
                         check=True).stdout.decode().splitlines()
    assert len(out) == len(vals)
    bad = [(v, g, _ref_line(ref, ids[k % 3].replace("\n", ""), v))
           for k, (v, g) in enumerate(zip(vals, out))
           if g != _ref_line(ref, ids[k % 3].replace("\n", ""), v)]
    assert not bad, bad[:5]
