"""ctypes mirror of include/omni_dev.h (device backend C ABI).

Thin plumbing for tests and bench.py: every compute call goes to
libomni_dev.so; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from ._native import check, dev_lib

THINKER, TALKER, DIT = 0, 1, 2
PREFILL, DECODE = 0, 1


class ModelDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "kind", "d_model", "n_layers", "n_heads", "n_kv_heads", "head_dim", "d_ff", "vocab",
        "cond_dim", "dit_channels", "dit_samples", "dit_steps")]


class StageLimits(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "max_batch_tokens", "max_resident", "max_seq_len", "kv_pages", "dit_max_tokens")]


class ArBatch(C.Structure):
    _fields_ = [("n_entries", C.c_int32),
                ("seq_id", C.POINTER(C.c_uint64)),
                ("phase", C.POINTER(C.c_int32)),
                ("span", C.POINTER(C.c_int32)),
                ("pos0", C.POINTER(C.c_int32)),
                ("out_index", C.POINTER(C.c_int32)),
                ("tokens", C.POINTER(C.c_int32)),
                ("cond_src", C.POINTER(C.c_uint64)),
                ("cond_row", C.POINTER(C.c_int32))]


class DitBatch(C.Structure):
    _fields_ = [("n_jobs", C.c_int32),
                ("request_id", C.POINTER(C.c_uint64)),
                ("token_offset", C.POINTER(C.c_int32)),
                ("n_tokens", C.POINTER(C.c_int32)),
                ("tokens", C.POINTER(C.c_int32))]


def _p(arr: np.ndarray, ct):
    return arr.ctypes.data_as(C.POINTER(ct))


def model_default(kind: int, **overrides) -> ModelDesc:
    m = ModelDesc()
    check(dev_lib().omni_model_default(kind, C.byref(m)))
    for k, v in overrides.items():
        setattr(m, k, v)
    return m


class Stage:
    """One model instance on one GPU (omni_stage*)."""

    def __init__(self, model: ModelDesc, limits: StageLimits | None = None, dev: int = 0,
                 seed: int = 1234):
        self.lib = dev_lib()
        self.model = model
        self.limits = limits or StageLimits(256, 64, 512, 0, 512)
        self.h = C.c_void_p()
        check(self.lib.omni_stage_create(C.byref(model), C.byref(self.limits), dev,
                                         C.c_uint64(seed), C.byref(self.h)))
        self._keep = []

    def close(self):
        if self.h:
            check(self.lib.omni_stage_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tensor(self, name: str) -> tuple[int, int, int]:
        p, r, c = C.c_uint64(), C.c_int64(), C.c_int64()
        check(self.lib.omni_stage_tensor(self.h, name.encode(), C.byref(p), C.byref(r), C.byref(c)))
        return p.value, r.value, c.value

    def set_sampling(self, top_k: int, seed: int = 0) -> None:
        """Greedy (top_k <= 1) or top-k sampling of decode rows (omni_stage_set_sampling)."""
        check(self.lib.omni_stage_set_sampling(self.h, top_k, C.c_uint64(seed)))

    def reserve_prompt(self, seq_id: int, pos0: int, tokens) -> None:
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        check(self.lib.omni_seq_reserve_prompt(self.h, C.c_uint64(seq_id), pos0, len(t), _p(t, C.c_int32)))

    def set_prefix_cache(self, enable: bool) -> None:
        check(self.lib.omni_stage_set_prefix_cache(self.h, 1 if enable else 0))

    def prefix_stats(self) -> dict:
        h, c, e = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(self.lib.omni_stage_prefix_stats(self.h, C.byref(h), C.byref(c), C.byref(e)))
        return {"hit_tokens": h.value, "cached_pages": c.value, "evicted_pages": e.value}

    def set_sm_share(self, sms: int) -> None:
        """SMs a DiT stage's persistent iteration may hold (<= 0: all; omni_stage_set_sm_share)."""
        check(self.lib.omni_stage_set_sm_share(self.h, sms))

    def reserve(self, seq_id: int, upto_tokens: int) -> None:
        check(self.lib.omni_seq_reserve(self.h, C.c_uint64(seq_id), upto_tokens))

    def after_pack(self, producer: "Stage") -> None:
        """This stage's next step waits for the producer's last connector pack."""
        check(self.lib.omni_stage_after_pack(self.h, producer.h))

    def weight_bytes(self) -> int:
        b = C.c_uint64()
        check(self.lib.omni_stage_weight_bytes(self.h, C.byref(b)))
        return b.value

    def ar_step(self, seq_id: Sequence[int], phase: Sequence[int], span: Sequence[int],
                pos0: Sequence[int], out_index: Sequence[int], tokens: Sequence[int],
                cond_src: Sequence[int] | None = None, cond_row: Sequence[int] | None = None,
                wait: bool = True):
        n = len(seq_id)
        arrs = dict(
            seq_id=np.ascontiguousarray(seq_id, dtype=np.uint64),
            phase=np.ascontiguousarray(phase, dtype=np.int32),
            span=np.ascontiguousarray(span, dtype=np.int32),
            pos0=np.ascontiguousarray(pos0, dtype=np.int32),
            out_index=np.ascontiguousarray(out_index, dtype=np.int32),
            tokens=np.ascontiguousarray(tokens, dtype=np.int32))
        b = ArBatch()
        b.n_entries = n
        b.seq_id = _p(arrs["seq_id"], C.c_uint64)
        for k in ("phase", "span", "pos0", "out_index", "tokens"):
            setattr(b, k, _p(arrs[k], C.c_int32))
        if cond_src is not None:
            arrs["cond_src"] = np.ascontiguousarray(cond_src, dtype=np.uint64)
            b.cond_src = _p(arrs["cond_src"], C.c_uint64)
        if cond_row is not None:
            arrs["cond_row"] = np.ascontiguousarray(cond_row, dtype=np.int32)
            b.cond_row = _p(arrs["cond_row"], C.c_int32)
        tok = np.full(n, -7, dtype=np.int32)
        margin = np.zeros(n, dtype=np.float32)
        check(self.lib.omni_ar_step(self.h, C.byref(b), _p(tok, C.c_int32), _p(margin, C.c_float)))
        self._keep = [arrs, b, tok, margin]
        if wait:
            self.wait()
        return tok, margin

    def dit_step(self, request_id, token_offset, n_tokens, tokens, wait: bool = True):
        arrs = dict(rid=np.ascontiguousarray(request_id, dtype=np.uint64),
                    off=np.ascontiguousarray(token_offset, dtype=np.int32),
                    nt=np.ascontiguousarray(n_tokens, dtype=np.int32),
                    tok=np.ascontiguousarray(tokens, dtype=np.int32))
        b = DitBatch(len(arrs["rid"]), _p(arrs["rid"], C.c_uint64), _p(arrs["off"], C.c_int32),
                     _p(arrs["nt"], C.c_int32), _p(arrs["tok"], C.c_int32))
        out = np.zeros(int(arrs["nt"].sum()) * 16, dtype=np.int32)
        check(self.lib.omni_dit_step(self.h, C.byref(b), _p(out, C.c_int32)))
        self._keep = [arrs, b, out]
        if wait:
            self.wait()
        return out

    def wait(self):
        check(self.lib.omni_stage_wait(self.h))

    def query(self) -> bool:
        rc = self.lib.omni_stage_query(self.h)
        if rc == 1:
            return False
        check(rc)
        return True

    def last_step_us(self) -> float:
        f = C.c_float()
        check(self.lib.omni_stage_last_step_us(self.h, C.byref(f)))
        return f.value

    def release(self, seq_id: int):
        check(self.lib.omni_seq_release(self.h, C.c_uint64(seq_id)))

    def hidden_row(self, seq_id: int, index: int) -> int:
        p = C.c_uint64()
        check(self.lib.omni_seq_hidden_row(self.h, C.c_uint64(seq_id), index, C.byref(p)))
        return p.value

    def pack_hidden(self, seq_id, begin, end, tokens, dst_base: int, dst_offset):
        a = dict(seq=np.ascontiguousarray(seq_id, dtype=np.uint64),
                 b=np.ascontiguousarray(begin, dtype=np.int32),
                 e=np.ascontiguousarray(end, dtype=np.int32),
                 t=np.ascontiguousarray(tokens, dtype=np.int32),
                 o=np.ascontiguousarray(dst_offset, dtype=np.uint64))
        check(self.lib.omni_pack_hidden(self.h, len(a["seq"]), _p(a["seq"], C.c_uint64),
                                        _p(a["b"], C.c_int32), _p(a["e"], C.c_int32),
                                        _p(a["t"], C.c_int32), C.c_uint64(dst_base),
                                        _p(a["o"], C.c_uint64)))
        self._keep = [a]


def pack_bytes(rows: int, d: int) -> int:
    lib = dev_lib()
    lib.omni_pack_bytes.restype = C.c_uint64
    return int(lib.omni_pack_bytes(rows, d))


# ---- plumbing: device memory (tests / bench) ------------------------------
def mem_alloc(nbytes: int, dev: int = 0) -> int:
    p = C.c_uint64()
    check(dev_lib().omni_mem_alloc(dev, C.c_uint64(nbytes), C.byref(p)))
    return p.value


def mem_free(ptr: int) -> None:
    check(dev_lib().omni_mem_free(C.c_uint64(ptr)))


def h2d(ptr: int, arr: np.ndarray) -> None:
    a = np.ascontiguousarray(arr)
    check(dev_lib().omni_mem_h2d(C.c_uint64(ptr), a.ctypes.data_as(C.c_void_p), C.c_uint64(a.nbytes)))


def d2h(ptr: int, shape, dtype) -> np.ndarray:
    out = np.empty(shape, dtype=dtype)
    check(dev_lib().omni_mem_d2h(out.ctypes.data_as(C.c_void_p), C.c_uint64(ptr), C.c_uint64(out.nbytes)))
    return out


def mem_set(ptr: int, byte: int, nbytes: int) -> None:
    check(dev_lib().omni_mem_set(C.c_uint64(ptr), byte, C.c_uint64(nbytes)))


def sync() -> None:
    check(dev_lib().omni_device_sync())
