"""Connector / control-frame conformance of libomni_serve (CPU).

Compiles tests/native/connector_conformance.cpp against the product's
control-plane headers and libomni_serve.so and runs it. The C++ file restates
the reference's own Catch2 cases (test_connector.cpp:31-170,
acceptance.cpp:194-266, test_payload_context.cpp:17-164) for host payloads
and for the DEVICE transport (locators of blobs in HBM, carried as encoded
DEVICE control frames)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_2602_02204_b200"
SRC = ROOT / "tests" / "native" / "connector_conformance.cpp"
OUT = PKG / "_build" / "tests" / "connector_conformance"


@pytest.fixture(scope="module")
def binary():
    from paper_2602_02204_b200 import build
    build.build()  # incremental: rebuilds the libraries only if a source changed
    OUT.parent.mkdir(parents=True, exist_ok=True)
    if not OUT.exists() or OUT.stat().st_mtime < max(SRC.stat().st_mtime, (PKG / "libomni_serve.so").stat().st_mtime):
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(PKG / "csrc" / "serve"), str(SRC), "-o", str(OUT),
                        "-L", str(PKG), "-lomni_serve", f"-Wl,-rpath,{PKG}", "-lpthread"], check=True)
    return OUT


def test_connector_and_control_frame_conformance(binary):
    r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    last = r.stdout.strip().splitlines()[-1]
    assert last.startswith("ALL OK"), last
    # every case ran in both host and DEVICE modes
    assert r.stdout.count("[device]") == r.stdout.count("[host]") >= 13
