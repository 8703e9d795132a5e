"""ctypes loader for the in-tree native libraries. Fails loudly when missing."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
_dev = None
_serve = None

STATUS = {0: "OK", 1: "EAGAIN", 2: "E_OOM", 3: "E_BADARG", 4: "E_FORWARD",
          5: "E_TRANSPORT", 6: "E_CUDA", 7: "E_NOGPU"}


class OmniError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def _load(name: str) -> C.CDLL:
    path = PKG / name
    if not path.exists():
        raise ImportError(f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    return C.CDLL(str(path), mode=C.RTLD_GLOBAL)


def dev_lib() -> C.CDLL:
    global _dev
    if _dev is None:
        lib = _load("libomni_dev.so")
        lib.omni_last_error.restype = C.c_char_p
        if hasattr(lib, 'omni_pack_bytes'):
            lib.omni_pack_bytes.restype = C.c_uint64
        _dev = lib
    return _dev


def serve_lib() -> C.CDLL:
    global _serve
    if _serve is None:
        dev_lib()
        lib = _load("libomni_serve.so")
        lib.omni_serve_last_error.restype = C.c_char_p
        _serve = lib
    return _serve


def check(status: int, lib: C.CDLL | None = None) -> None:
    if status != 0:
        lib = lib or dev_lib()
        # the serve library re-exports libomni_dev's symbols (dlsym searches
        # its dependencies), so pick its own error getter first
        if hasattr(lib, "omni_serve_last_error"):
            getter = lib.omni_serve_last_error
        else:
            getter = lib.omni_last_error
        getter.restype = C.c_char_p
        raise OmniError(status, (getter() or b"").decode())
