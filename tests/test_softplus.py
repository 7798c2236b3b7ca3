"""The device log_add (csrc/softplus.cuh, branch-free table-driven fp64)
compiled for the host and checked against 40-digit values: softplus within
3 ulp, and log_add bit-identical to glibc in >= 97% of draws (the rest are
1-ulp roundings in the non-plateau regime)."""
import math
import os
import random
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def spc(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("sp") / "spc")
    subprocess.run(["g++", "-O2", "-std=c++17", "-o", exe,
                    os.path.join(ROOT, "tests", "cpp", "softplus_check.cpp")], check=True)
    return exe


def run(spc, pairs):
    inp = "\n".join(f"{a!r} {b!r}" for a, b in pairs)
    out = subprocess.run([spc], input=inp, capture_output=True, text=True).stdout.split()
    return [tuple(float.fromhex(out[4 * i + k]) for k in range(4)) for i in range(len(pairs))]


def test_softplus_accuracy(spc):
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 40
    rng = random.Random(7)
    pairs = []
    for _ in range(4000):
        a = -rng.uniform(0, 2000) * rng.choice([1, 0.01])
        d = -rng.choice([rng.uniform(0, 1), rng.uniform(0, 40), rng.uniform(0, 700),
                         10 ** rng.uniform(-12, 0)])
        pairs.append((a, a + d))
    worst = 0.0
    same = 0
    for (a, b), (sp, la, _, _) in zip(pairs, run(spc, pairs)):
        d = min(a, b) - max(a, b)
        ex = mp.log1p(mp.exp(mp.mpf(d)))
        worst = max(worst, float(abs((mp.mpf(sp) - ex) / ex)) / 2 ** -53)
        same += la == max(a, b) + math.log1p(math.exp(d))
    assert worst <= 3.0
    assert same >= 0.97 * len(pairs)


def test_log_add_zero_semantics(spc):
    """logmath.hpp:19-23: zero operands return the other bit-exactly."""
    res = run(spc, [(-1e30, -3.25), (-3.25, -1e30), (-1e30, -1e30),
                    (-1.0000000150474662e30, -1e30), (0.0, 0.0)])
    assert res[0][1] == -3.25 and res[1][1] == -3.25
    assert res[2][1] == -1e30 and res[3][1] == -1e30
    assert res[4][1] == math.log(2.0)


def test_exp_log_accuracy(spc):
    """exp_neg / log_pos (the two halves of the softplus, used for the
    contenders' parallel psi): within 3 ulp of 40-digit values."""
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 40
    rng = random.Random(11)
    pairs = [(0.0, -rng.choice([rng.uniform(0, 1), rng.uniform(0, 40), rng.uniform(0, 700),
                                10 ** rng.uniform(-12, 0)])) for _ in range(4000)]
    we = wl = 0.0
    for (_, d), (_, _, e, lg) in zip(pairs, run(spc, pairs)):
        ex = mp.exp(mp.mpf(d))
        if ex > mp.mpf(2) ** -1000:
            we = max(we, float(abs((mp.mpf(e) - ex) / ex)) / 2 ** -53)
        lx = mp.log(1 - mp.mpf(d))
        if lx > 0:
            wl = max(wl, float(abs(mp.mpf(lg) - lx) / max(lx, mp.mpf(1))) / 2 ** -53)
    assert we <= 3.0 and wl <= 3.0, (we, wl)
    z = run(spc, [(0.0, 0.0), (0.0, -1e30)])
    assert z[0][2] == 1.0 and z[0][3] == 0.0 and z[1][2] == 0.0
