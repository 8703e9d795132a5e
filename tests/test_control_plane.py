"""Bit-exact parity of the B200 build's C++ control plane (libomni_serve)
against the UNMODIFIED reference, on CPU.

tests/golden/ holds traces produced by oracle/ref_harness (the reference
headers compiled as-is, oracle/make_golden.sh). oracle/mock_pipeline.cpp
restates the reference's mock hooks as plugins of the NEW control plane and
prints the same trace: every prefill / decode hook call with its virtual-clock
instant (= batch membership per iteration), every packed chunk with its
payload digest (= chunk cuts + wire layout), and every request's outputs and
metrics timeline (= routing, JCT/TTFT). Equality of the full text proves
ar_engine.hpp:66-374, diffusion_engine.hpp:75-128, orchestrator.hpp:377-734,
connector streams and the bench workload are reproduced bit-for-bit.
"""
import ctypes as C
import gzip
import json
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden"
MOCK = ROOT / "oracle" / "_build" / "liboracle_mock.so"


@pytest.fixture(scope="module")
def mock():
    import subprocess  # make: rebuilds when libomni_serve.so or its headers changed
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "_build/liboracle_mock.so"], check=True)
    lib = C.CDLL(str(MOCK))
    lib.oracle_mock_trace.restype = C.c_long
    lib.oracle_mock_trace.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                      C.c_char_p, C.c_size_t]
    lib.oracle_mock_csv.restype = C.c_long
    lib.oracle_mock_csv.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_char_p, C.c_size_t]
    lib.oracle_workload_digest.restype = C.c_uint64
    lib.oracle_workload_digest.argtypes = [C.c_uint64, C.c_uint64]
    return lib


def run_trace(lib, cfg, n, seed, conc, stream, c0=0, c1=0):
    text = (ROOT / "configs" / cfg).read_text().encode()
    cap = 64 << 20
    buf = C.create_string_buffer(cap)
    k = lib.oracle_mock_trace(text, n, seed, conc, stream, c0, c1, buf, cap)
    assert k >= 0, buf.value.decode()
    return buf.value.decode()


def cases():
    out = []
    for line in (GOLD / "traces.index").read_text().splitlines():
        f = line.split()
        if f:
            out.append(f)
    return out


def fnv(data: bytes) -> str:
    h = 1469598103934665603
    for b in data:
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


@pytest.mark.parametrize("case", cases(), ids=lambda c: c[0])
def test_trace_bit_exact(mock, case):
    name, cfg, n, seed, conc, stream, *chunks = case
    c0, c1 = (int(chunks[0]), int(chunks[1])) if chunks else (0, 0)
    got = run_trace(mock, cfg, int(n), int(seed), int(conc), int(stream), c0, c1)
    want = gzip.decompress((GOLD / f"trace_{name}.txt.gz").read_bytes()).decode()
    if got != want:
        g, w = got.splitlines(), want.splitlines()
        for i, (a, b) in enumerate(zip(g, w)):
            assert a == b, f"first divergence at line {i}:\n new: {a}\n ref: {b}"
        assert len(g) == len(w), f"line count {len(g)} vs {len(w)}"


def test_digests_match_reference(mock):
    d = json.loads((GOLD / "digests.json").read_text())
    assert f"{mock.oracle_workload_digest(100, 7):016x}" == d["workload_digest"]
    text = (ROOT / "configs" / "omni3.json").read_text().encode()
    buf = C.create_string_buffer(1 << 20)
    k = mock.oracle_mock_csv(text, 100, 7, 16, buf, 1 << 20)
    assert k == d["disagg_csv_len"], buf.value[:200]
    assert fnv(buf.value) == d["disagg_csv_digest"]
