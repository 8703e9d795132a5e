"""Multi-process stage placement over CUDA IPC.

tests/native/ipc_placement.cpp forks a producer (Thinker) and a consumer
(Talker) process. `cpu`: the cross-process control plane (HANDOFF of the
arena / event handles, DEVICE CHUNK_NOTICE / EOS frames, ACKs, receiver-side
protocol checks, peer loss) on synthetic locators. `gpu`: the Thinker packs
into the consumer's IPC-imported arena, ordered by an interprocess event; the
consumer checks the blobs bit-exact against the in-process pack and the
Talker's tokens / margins bit-identical when fed from the IPC arena."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_2602_02204_b200"
SRC = ROOT / "tests" / "native" / "ipc_placement.cpp"
OUT = PKG / "_build" / "tests" / "ipc_placement"


@pytest.fixture(scope="module")
def binary():
    if not (PKG / "libomni_serve.so").exists():
        from paper_2602_02204_b200 import build
        build.build()
    OUT.parent.mkdir(parents=True, exist_ok=True)
    if not OUT.exists() or OUT.stat().st_mtime < max(SRC.stat().st_mtime, (PKG / "libomni_serve.so").stat().st_mtime):
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(PKG / "csrc" / "serve"), "-I", str(ROOT / "include"),
                        str(SRC), "-o", str(OUT), "-L", str(PKG), "-lomni_serve", "-lomni_dev",
                        f"-Wl,-rpath,{PKG}", "-lpthread"], check=True)
    return OUT


def _run(binary, mode):
    r = subprocess.run([str(binary), mode], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.strip().splitlines()[-1] == "ALL OK", r.stdout
    return r.stdout


def test_ipc_control_plane_across_processes(binary):
    out = _run(binary, "cpu")
    assert "receiver rejects" in out and "TransportDown" in out


@pytest.mark.gpu
def test_thinker_to_talker_across_processes_cuda_ipc(binary):
    out = _run(binary, "gpu")
    assert "bit-exact with the in-process pack" in out and "bit-identical" in out
