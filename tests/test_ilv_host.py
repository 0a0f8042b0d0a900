"""K_ilv's ring length (kernels.cu, DESIGN.md V.2): the round structure of the
kernel, replayed on the host (tests/native/ilv_rounds.cpp), never lets a
producer run more than P/2 + 1 table positions ahead of the position its
consumer reads, for every depth P <= 64, v <= 8 chunks and m in {P, 2P, 3P}
micro-batches (the lead does not depend on durations: a round runs every op
whose input exists).  The kernel's rings hold Q >= P/2 + 2 entries, so no
unread entry is overwritten; it also checks this at run time (status -5)."""
import ctypes as C
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "ilv_rounds.cpp")


@pytest.fixture(scope="module")
def lead(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("ilv") / "ilv_rounds.so")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", SRC, "-o", out])
    lib = C.CDLL(out)
    lib.ilv_max_lead.restype = C.c_int
    lib.ilv_max_lead.argtypes = [C.c_int] * 3
    return lib.ilv_max_lead


def ring_len(P):  # the host's choice in run_phases (kernels.cu)
    q = 4
    while q < P // 2 + 2:
        q *= 2
    return q


def test_ring_never_overwrites_unread(lead):
    worst = {}
    for P in range(2, 65):
        for v in range(2, 9):
            for m in (P, 2 * P, 3 * P):
                x = lead(P, v, m)
                assert x >= 0, ("deadlock", P, v, m)
                worst[P] = max(worst.get(P, 0), x)
        assert worst[P] <= P // 2 + 1, (P, worst[P])
        assert worst[P] < ring_len(P)
