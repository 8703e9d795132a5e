"""ctypes mirror of include/omni_serve.h (pipeline-level C ABI)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, fields

from ._native import check, serve_lib


class PipelineOpts(C.Structure):
    _fields_ = [("weight_seed", C.c_uint64), ("small_models", C.c_int32), ("device", C.c_int32)]


class BenchSpec(C.Structure):
    _fields_ = [("n", C.c_uint64), ("seed", C.c_uint64), ("concurrency", C.c_uint64),
                ("stream", C.c_int32), ("poisson", C.c_int32), ("rate", C.c_double),
                ("prompt_min", C.c_uint32), ("prompt_max", C.c_uint32), ("clock", C.c_char_p),
                ("trace", C.c_int32), ("talker_chunk", C.c_int32), ("vocoder_chunk", C.c_int32),
                ("capture", C.c_int32)]


class BenchResult(C.Structure):
    _fields_ = [("completed", C.c_uint64), ("failed", C.c_uint64),
                ("makespan_us", C.c_double), ("requests_per_s", C.c_double),
                ("mean_jct_us", C.c_double), ("p50_jct_us", C.c_double), ("p95_jct_us", C.c_double),
                ("p99_jct_us", C.c_double), ("mean_ttft_us", C.c_double), ("p99_ttft_us", C.c_double),
                ("mean_rtf", C.c_double), ("text_tokens", C.c_uint64), ("codec_tokens", C.c_uint64),
                ("wave_samples", C.c_uint64), ("dev_ms_thinker", C.c_double), ("dev_ms_talker", C.c_double),
                ("dev_ms_dit", C.c_double), ("steps_thinker", C.c_uint64), ("steps_talker", C.c_uint64),
                ("steps_dit", C.c_uint64), ("output_digest", C.c_uint64), ("preemptions", C.c_uint64),
                ("wall_s", C.c_double),
                ("host_ms_thinker", C.c_double), ("host_ms_talker", C.c_double), ("host_ms_dit", C.c_double),
                ("gap_us_thinker", C.c_double), ("gap_us_talker", C.c_double), ("gap_us_dit", C.c_double)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class Pipeline:
    """A B200 stage pipeline built from a reference-format deployment config."""

    def __init__(self, config_json: str, weight_seed: int = 1234, small_models: bool = False, device: int = 0):
        self.lib = serve_lib()
        self.h = C.c_void_p()
        opts = PipelineOpts(weight_seed, 1 if small_models else 0, device)
        check(self.lib.omni_pipeline_create(config_json.encode(), C.byref(opts), C.byref(self.h)), self.lib)

    def close(self):
        if self.h:
            check(self.lib.omni_pipeline_destroy(self.h), self.lib)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bench(self, n=100, seed=7, concurrency=16, stream=True, clock="device", trace=False,
              poisson=False, rate=1.0, talker_chunk=0, vocoder_chunk=0, capture=False) -> dict:
        spec = BenchSpec(n, seed, concurrency, 1 if stream else 0, 1 if poisson else 0, rate, 0, 0,
                         clock.encode(), 1 if trace else 0, talker_chunk, vocoder_chunk, 1 if capture else 0)
        res = BenchResult()
        check(self.lib.omni_pipeline_bench(self.h, C.byref(spec), C.byref(res)), self.lib)
        return res.as_dict()

    def serve_start(self, listen: str = "127.0.0.1:0") -> int:
        """Live serving: orchestrator loop (device clock) + HTTP front end; returns the port."""
        port = C.c_int32()
        check(self.lib.omni_pipeline_serve_start(self.h, listen.encode(), C.byref(port)), self.lib)
        return port.value

    def serve_stop(self) -> None:
        check(self.lib.omni_pipeline_serve_stop(self.h), self.lib)

    def output(self, request_id: int, what: int):
        """Per-request output of the last bench(capture=True) run (OMNI_OUT_*)."""
        import numpy as np
        f = self.lib.omni_pipeline_output
        f.restype = C.c_size_t
        f.argtypes = [C.c_void_p, C.c_uint64, C.c_int32, C.c_void_p, C.c_size_t]
        n = f(self.h, request_id, what, None, 0)
        dt = {0: np.uint8, 1: np.int32, 2: np.int32, 3: np.int32, 4: np.uint16}[what]
        out = np.empty(n // np.dtype(dt).itemsize, dtype=dt)
        if n:
            f(self.h, request_id, what, out.ctypes.data, n)
        return out

    def text(self, what: int) -> str:
        self.lib.omni_pipeline_text.restype = C.c_size_t
        n = self.lib.omni_pipeline_text(self.h, what, None, 0)
        buf = C.create_string_buffer(n + 1)
        self.lib.omni_pipeline_text(self.h, what, buf, n + 1)
        return buf.value.decode()

    def csv(self) -> str:
        return self.text(0)

    def trace(self) -> str:
        return self.text(1)
