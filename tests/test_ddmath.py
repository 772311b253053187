"""CPU suite: the double-double log/sin/cos of the device generators
(csrc/ddmath.cuh, compiled here for the host by tests/helpers/ddmath_driver.cpp)
are correctly rounded, and the moons they produce are the host generator's
(proj/src/datasets.cpp:32-55 restated in csrc/datasets.cpp) to the last bit
after rounding to fp32. The device kernels run the same header; their own
outputs are compared with the host generators in test_gpu_generators.py."""
import os
import subprocess
from decimal import Decimal, getcontext

import numpy as np
import pytest

from paper_2310_13870_b200 import datasets

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
getcontext().prec = 60
PI = Decimal("3.14159265358979323846264338327950288419716939937510582097494459")


@pytest.fixture(scope="module")
def driver(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("dd") / "ddmath_driver")
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off",
                    "-I", os.path.join(ROOT, "paper_2310_13870_b200", "csrc"),
                    os.path.join(ROOT, "tests", "helpers", "ddmath_driver.cpp"), "-o", exe],
                   check=True)
    return exe


def run(exe, mode, xs):
    out = subprocess.run([exe, mode], input="\n".join(float(x).hex() for x in xs),
                         capture_output=True, text=True, check=True).stdout.split()
    return np.array([float.fromhex(v) for v in out])


def dec_sin_cos(x: float):
    r = Decimal(x) % (2 * PI)
    s, c, term_s, term_c, k = Decimal(0), Decimal(0), r, Decimal(1), 0
    while abs(term_s) > Decimal(10) ** -58 or abs(term_c) > Decimal(10) ** -58:
        s += term_s
        c += term_c
        term_s = -term_s * r * r / ((2 * k + 2) * (2 * k + 3))
        term_c = -term_c * r * r / ((2 * k + 1) * (2 * k + 2))
        k += 1
    return float(s), float(c)  # float(Decimal) rounds correctly


def test_log_correctly_rounded(driver):
    rng = np.random.default_rng(3)
    # Box-Muller's arguments (k 2^-53) plus a spread of magnitudes
    xs = list((rng.integers(1, 2 ** 53, 1500) * 2.0 ** -53))
    xs += list(np.exp(rng.uniform(-700, 700, 500)))
    xs += [2.0 ** -53, 0.5, 1.0, 2.0, np.nextafter(1.0, 0), np.nextafter(1.0, 2), 5e-324]
    got = run(driver, "log", xs)
    want = np.array([float(Decimal(x).ln()) for x in xs])
    assert np.array_equal(got, want)


def test_sin_cos_correctly_rounded(driver):
    rng = np.random.default_rng(4)
    xs = list(6.283185307179586476925286766559 * (rng.integers(0, 2 ** 53, 1000) * 2.0 ** -53))
    n = 500_000  # the moons' arcs t = pi i / (n - 1)
    xs += [3.14159265358979323846 * i / (n - 1) for i in rng.integers(0, n, 500)]
    xs += [0.0, np.pi / 2, np.pi, 3 * np.pi / 2, 2 * np.pi, np.pi / 4, 1e-10, 7.5]
    s, c = run(driver, "sin", xs), run(driver, "cos", xs)
    want = [dec_sin_cos(x) for x in xs]
    assert np.array_equal(s, np.array([w[0] for w in want]))
    assert np.array_equal(c, np.array([w[1] for w in want]))


def test_glibc_differs_in_rare_last_bits_only(driver):
    # glibc's log/sin/cos are within 0.502 ulp, not always correctly rounded:
    # the documented reason the device's fp64 coordinates may differ in the
    # last bit (include/fsgg.h). Measured here: ~0.1% of arguments.
    N = 200_000
    out = subprocess.run([driver, "glibc", str(N)], capture_output=True, text=True,
                         check=True).stdout.split()
    bl, bs, bc = (int(v) for v in out)
    for count in (bl, bs, bc):
        assert count < 0.005 * N


def test_dd_moons_round_to_the_host_generator_fp32(driver):
    # C3's inputs: the dd-math moons equal the host generator's fp64 except in
    # rare last bits, and are identical once rounded to fp32
    n = 1_000_000
    raw = subprocess.run([driver, "moons", str(n), "0.05", "1"], capture_output=True,
                         check=True).stdout
    dd = np.frombuffer(raw, np.float64).reshape(n, 2)
    host, _ = datasets.make_moons(n, 0.05, 1)
    assert np.array_equal(dd.astype(np.float32), host.astype(np.float32))
    diff = dd != host
    assert diff.mean() < 0.005
    # absolute: a last-bit difference in cos/sin (|value| <= 1) or in a noise
    # term; relative ulps blow up where 1 - cos(t) or the noise cancels
    assert np.abs(dd - host).max() <= 4 * np.spacing(1.0)
