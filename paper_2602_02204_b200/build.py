"""In-tree build of the native libraries (sm_100a only).

    libomni_dev.so   — CUDA kernels + device runtime, C-ABI include/omni_dev.h
    libomni_serve.so — C++ stage-graph control plane (API mirror of the
                       reference's omniserve headers) + the GPU stage plugins,
                       C-ABI include/omni_serve.h; links libomni_dev.so

Objects go to paper_2602_02204_b200/_build/, the .so files next to this file
(git-ignored, but they travel to the GPU box with the gpurun snapshot).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "g++"  # PATH g++ (an env CXX wrapper in this image drops libstdc++)
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

DEV_LIB = PKG / "libomni_dev.so"
SERVE_LIB = PKG / "libomni_serve.so"


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def _deps_newer(obj: Path, src: Path, headers: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(h.stat().st_mtime > t for h in headers)


def _compile(src: Path, obj: Path, headers: list[Path], extra: list[str]) -> Path:
    if not _deps_newer(obj, src, headers):
        return obj
    obj.parent.mkdir(parents=True, exist_ok=True)
    inc = ["-I", str(ROOT / "include"), "-I", str(CSRC / "dev"), "-I", str(CSRC / "serve"),
           "-I", JSON_INC]
    if src.suffix == ".cu":
        cmd = [NVCC, *ARCH, "-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v" if os.environ.get("OMNI_PTXAS_V") else "-O3",
               "--expt-relaxed-constexpr", *inc, *extra, "-c", str(src), "-o", str(obj)]
    else:
        cmd = [CXX, "-std=c++20", "-O2", "-g", "-fPIC", "-Wall", "-Wno-unused-function",
               "-I", f"{CUDA_HOME}/include", *inc, *extra, "-c", str(src), "-o", str(obj)]
    _run(cmd)
    return obj


def _build_lib(name: str, srcdir: Path, out: Path, link: list[str], jobs: int) -> Path:
    srcs = sorted([*srcdir.glob("*.cu"), *srcdir.glob("*.cpp")])
    headers = sorted([*(CSRC / "dev").glob("*.h"), *(CSRC / "dev").glob("*.cuh"),
                      *(CSRC / "serve").glob("*.h"), *(CSRC / "serve").glob("*.hpp"),
                      *(CSRC / "serve" / "omni").glob("*.hpp"),
                      *(ROOT / "include").glob("*.h")])
    objs_dir = BUILD / name
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        futs = [ex.submit(_compile, s, objs_dir / (s.name + ".o"), headers, []) for s in srcs]
        objs = [f.result() for f in futs]
    newest = max(o.stat().st_mtime for o in objs)
    if not out.exists() or out.stat().st_mtime < newest:
        _run([NVCC, *ARCH, "-shared", "-o", str(out), *map(str, objs), *link])
    return out


def build(jobs: int | None = None) -> tuple[Path, Path]:
    jobs = jobs or max(2, os.cpu_count() or 2)
    dev = _build_lib("dev", CSRC / "dev", DEV_LIB, ["-lcudart"], jobs)
    serve = _build_lib("serve", CSRC / "serve", SERVE_LIB,
                       ["-L", str(PKG), "-lomni_dev", "-Xlinker", "-rpath,$ORIGIN", "-lcudart",
                        "-lpthread"], jobs)
    return dev, serve


if __name__ == "__main__":
    d, s = build()
    print(d, s, file=sys.stderr)
