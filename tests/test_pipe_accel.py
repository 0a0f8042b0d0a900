"""The product's 1F1B recurrence with its exact steady-regime jumps (Pipe<P>,
hsim_core.cuh; DESIGN.md §5 "1F1B acceleration"), compiled for the host by a
test harness, against the oracle's event-driven pipeline (oracle.pipeline,
DESIGN.md C.7) on stress inputs: balanced stages of nearly equal speed (long
transients, the affine regime), cyclic regimes, tiny and huge m, large p2p
costs.  CPU only; the GPU parity tests run the same code on the device."""
import ctypes as C
import os
import random
import subprocess

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "pipe_host.cpp")
HDR = os.path.join(ROOT, "paper_2508_05370_b200", "csrc", "hsim_core.cuh")


@pytest.fixture(scope="module")
def host(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("pipe") / "pipe_host.so")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC", SRC, "-o", out])
    lib = C.CDLL(out)
    lib.pipe_host_run.restype = C.c_int64
    lib.pipe_host_run.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]

    def run(f, g, c, m):
        P = len(f)
        fa, ga = (C.c_int64 * P)(*f), (C.c_int64 * P)(*g)
        ca = (C.c_int64 * max(P, 1))(*(list(c) + [0] * (P - len(c))))
        sk = C.c_int64(0)
        t = lib.pipe_host_run(P, m, fa, ga, ca, C.byref(sk))
        return t, sk.value
    return run


def _case(rng, P, noise, cscale):
    base = rng.randint(10 ** 5, 10 ** 8)
    f = [max(1, int(base * (1 + noise * rng.uniform(-1, 1)))) for _ in range(P)]
    g = [2 * x + rng.randint(0, 1000) for x in f]
    c = [rng.randint(0, max(1, base // cscale)) for _ in range(P - 1)]
    return f, g, c


@pytest.mark.parametrize("P", list(range(1, 17)))
def test_pipe_jumps_exact_random(host, P):
    rng = random.Random(0x5EED2508 + P)
    skipped = 0
    for trial in range(60):
        f, g, c = _case(rng, P, rng.choice([0.0, 1e-5, 1e-3, 1e-2, 0.1, 0.5]), rng.choice([3, 30, 1000, 10 ** 6]))
        m = rng.choice([1, 2, P - 1, P, P + 1, P + 3, P + 4, P + 5, 2 * P + 7, 64, 333, 1024, 2048])
        m = max(1, m)
        got, sk = host(f, g, c, m)
        assert got == oracle.pipeline(f, g, c, m), (P, m, f, g, c)
        skipped += sk
    if P >= 2:
        assert skipped > 0  # the jumps are exercised


def test_pipe_long_transient_config2_stage_times(host):
    # config-2 stage durations with two nearly equally fast stages (A100 /
    # H100 split 4/4/12/12 layers): a ~500-pair transient before cyclicity 1
    f = [111547127, 86725310, 111503970, 93608271]
    g = [223094245, 173450613, 223007931, 187216534]
    c = [223822 // 2, 223822 // 2, 223822 // 2]
    for m in (124, 258, 545, 1024, 4096):
        got, sk = host(f, g, c, m)
        assert got == oracle.pipeline(f, g, c, m)
        assert sk > (m - 4) // 2  # most steady pairs are jumped


def test_pipe_uniform_closed_form(host):
    # uniform stages, c = 0: (m + P - 1)(f + g) (BASELINE.json closed form)
    for P in (1, 2, 4, 8, 16):
        for m in (1, P, 100, 1000):
            got, _ = host([7] * P, [13] * P, [0] * (P - 1), m)
            assert got == (m + P - 1) * 20


def test_pipe_jumps_exact_small_integers(host):
    # small integer durations: many exact ties between competing operands
    rng = random.Random(7)
    for trial in range(4000):
        P = rng.choice([2, 3, 4, 5, 8, 12, 16])
        m = rng.choice([P + 4, 30, 100, 400])
        base = rng.randint(20, 2000)
        f = [base + rng.randint(-3, 3) for _ in range(P)]
        g = [base + rng.randint(-3, 3) for _ in range(P)]
        c = [rng.choice([0, 0, 1, 5, 50, base]) for _ in range(P - 1)]
        assert host(f, g, c, m)[0] == oracle.pipeline(f, g, c, m), (P, m, f, g, c)
