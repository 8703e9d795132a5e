"""ORACLE / TEST INFRASTRUCTURE: ctypes access to the CPU checkers.

  * liboracle_models.so (models_cpu.c): fp32 restatement of the stage models
  * _ref/ref_harness: the unmodified reference headers (golden traces)
  * plain-Python restatements of the reference's integer semantics
    (reference_pipeline.hpp:20-45, diffusion_engine.hpp:28-43, payload.hpp:142-166)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.
"""
from __future__ import annotations

import ctypes as C
import struct
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle_models.so"
REF = HERE / "_ref" / "ref_harness"


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE), "_build/liboracle_models.so"], check=True)
    if Path("/root/reference/proj/include").exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "_ref/ref_harness"], check=True)


class Desc(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("kind", "d", "L", "H", "KVH", "hd", "ff", "V", "cond_dim",
                                       "C", "S", "T")]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        L.om_create.restype = C.c_void_p
        L.om_create.argtypes = [C.POINTER(Desc), C.c_uint64]
        L.om_destroy.argtypes = [C.c_void_p]
        L.om_seq_new.restype = C.c_void_p
        L.om_seq_new.argtypes = [C.c_void_p, C.c_int]
        L.om_seq_free.argtypes = [C.c_void_p]
        L.om_ar_feed.restype = C.c_int
        L.om_ar_feed.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_int),
                                 C.POINTER(C.c_int), C.POINTER(C.c_uint16), C.c_int,
                                 C.POINTER(C.c_float), C.POINTER(C.c_uint16), C.POINTER(C.c_float)]
        L.om_dit_denoise.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int), C.POINTER(C.c_int32), C.POINTER(C.c_float)]
        L.om_weight_bits.restype = C.c_uint16
        L.om_weight_bits.argtypes = [C.c_void_p, C.c_char_p, C.c_int64, C.c_int64]
        _lib = L
    return _lib


def desc_from(model) -> Desc:
    """Maps an omni_model_desc (paper_2602_02204_b200.dev.ModelDesc) onto the oracle's."""
    return Desc(model.kind, model.d_model, model.n_layers, model.n_heads, model.n_kv_heads,
                model.head_dim, model.d_ff, model.vocab, model.cond_dim, model.dit_channels,
                model.dit_samples, model.dit_steps)


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


class Model:
    def __init__(self, model_desc, seed: int):
        self.d = desc_from(model_desc)
        self.h = lib().om_create(C.byref(self.d), C.c_uint64(seed))

    def __del__(self):
        if getattr(self, "h", None):
            lib().om_destroy(self.h)
            self.h = None

    def weight_bits(self, name: str, row: int, col: int) -> int:
        return int(lib().om_weight_bits(self.h, name.encode(), row, col))

    def new_seq(self, cap: int = 512) -> "Seq":
        return Seq(self, cap)

    def dit(self, rid, pos, ids, with_latents=False):
        n = len(ids)
        rid = np.ascontiguousarray(rid, dtype=np.uint64)
        pos = np.ascontiguousarray(pos, dtype=np.int32)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        out = np.zeros(n * self.d.S, dtype=np.int32)
        lat = np.zeros(n * self.d.S * self.d.C, dtype=np.float32) if with_latents else None
        lib().om_dit_denoise(self.h, n, rid.ctypes.data_as(C.POINTER(C.c_uint64)), _ip(pos), _ip(ids),
                             out.ctypes.data_as(C.POINTER(C.c_int32)),
                             lat.ctypes.data_as(C.POINTER(C.c_float)) if lat is not None else None)
        return (out, lat) if with_latents else out


class Seq:
    def __init__(self, model: Model, cap: int):
        self.m = model
        self.h = lib().om_seq_new(model.h, cap)

    def __del__(self):
        if getattr(self, "h", None):
            lib().om_seq_free(self.h)
            self.h = None

    def feed(self, tokens, decode: bool, cond_rows=None, hid_rows=None):
        """Returns (token, logits, hidden_bits, margin) for decode, else None."""
        n = len(tokens)
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        cr = np.ascontiguousarray(cond_rows if cond_rows is not None else [0] * n, dtype=np.int32)
        hr = None if hid_rows is None else np.ascontiguousarray(hid_rows, dtype=np.uint16)
        V, d = self.m.d.V, self.m.d.d
        lg = np.zeros(V, dtype=np.float32)
        hid = np.zeros(d, dtype=np.uint16)
        mg = C.c_float()
        tok = lib().om_ar_feed(self.m.h, self.h, n, _ip(t), _ip(cr),
                               hr.ctypes.data_as(C.POINTER(C.c_uint16)) if hr is not None else None,
                               1 if decode else 0, lg.ctypes.data_as(C.POINTER(C.c_float)),
                               hid.ctypes.data_as(C.POINTER(C.c_uint16)), C.byref(mg))
        if tok == -2:
            raise RuntimeError("oracle sequence capacity exceeded")
        return (tok, lg, hid, mg.value) if decode else None


# ---------------------------------------------------------------------------
# Reference integer semantics restated (used as known-answer checkers)
# ---------------------------------------------------------------------------
M32 = 0xFFFFFFFF


def mix(h: int, t: int) -> int:  # reference_pipeline.hpp:20-22
    return (h * 1000003 + t + 1) & M32


def fold_prompt(prompt, seed: int) -> int:  # reference_pipeline.hpp:24-28
    h = seed & M32
    for t in prompt:
        h = mix(h, t)
    return h


def target_length(h: int) -> int:  # reference_pipeline.hpp:30-32
    return (h % 64) + 1


def thinker_generate(prompt, seed):  # reference_pipeline.hpp:52-64
    h = fold_prompt(prompt, seed)
    toks, hid = [], []
    for step in range(target_length(h)):
        h = mix(h, step)
        toks.append(h % 255 + 1)
        hid.append([(h >> (4 * k)) & 0xF for k in range(8)])
    return toks, hid


def codec_token(t: int, hsum: int, i: int) -> int:  # reference_pipeline.hpp:43-45
    return (t * 7 + hsum + i) % 64


M64 = 0xFFFFFFFFFFFFFFFF


def talker_generate(text, hidden):  # reference_pipeline.hpp:66-75
    return [codec_token(t, sum(h), i) for t, h in zip(text, hidden) for i in range(4)]


def mix64(x: int) -> int:  # csrc/dev/rng.h mix64 (splitmix64 finaliser)
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def sample_hash(seed: int, key: int, index: int) -> int:  # csrc/dev/rng.h sample_hash
    return mix64(seed ^ mix64(((key << 32) ^ index ^ 0x73616D706C650000) & M64))


def denoise_closed_form(codec, S=16):  # diffusion_engine.hpp:28-43
    out = []
    for c in codec:
        for s in range(S):
            out.append(((c * (s + 1)) % 128) - 64)
    return out


def encode_payload(dtype: int, shape, body: bytes) -> bytes:  # payload.hpp:142-151
    return bytes([dtype, len(shape)]) + b"".join(struct.pack("<I", d) for d in shape) + body


def fnv1a(data: bytes, h: int = 1469598103934665603) -> int:  # connector.hpp:198-205
    for b in data:
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def pack_hidden_blob(tokens, hidden_rows_u16: np.ndarray) -> bytes:
    """FIX16 {n, 1+d} chunk: col 0 = token, cols 1..d = bf16 bits."""
    n, d = hidden_rows_u16.shape
    body = np.zeros((n, d + 1), dtype="<u2")
    body[:, 0] = np.asarray(tokens, dtype=np.uint16)
    body[:, 1:] = hidden_rows_u16
    return encode_payload(2, [n, d + 1], body.tobytes())
