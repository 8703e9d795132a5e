"""Streaming front end: the reference's test_http.cpp cases
(health, 400s, non-streaming and NDJSON streaming generate, aggregate
metrics) against the B200 build's HttpService (csrc/serve/http_service.cpp).

CPU: the control plane on the wall clock with the reference's mock hooks
(oracle/mock_pipeline.cpp), outputs checked against the oracle's restatement
of reference_pipeline.hpp (thinker_generate / codec_token / denoise). GPU: the
B200 pipeline (small models) behind omni_pipeline_serve_start; the streamed
chunks must reassemble to the non-streamed waveform of the same request."""
import base64
import ctypes as C
import http.client
import json
import struct
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
MOCK = ROOT / "oracle" / "_build" / "liboracle_mock.so"
CFG = (ROOT / "configs" / "omni3.json").read_text()


def b64_i32(s: str):
    b = base64.b64decode(s)
    return list(struct.unpack(f"<{len(b) // 4}i", b))


def call(port, method, path, body=None):
    c = http.client.HTTPConnection("127.0.0.1", port, timeout=120)
    c.request(method, path, body=None if body is None else (body if isinstance(body, str) else json.dumps(body)),
              headers={"Content-Type": "application/json"})
    r = c.getresponse()
    data = r.read().decode()
    c.close()
    return r.status, r.getheader("Content-Type"), data


@pytest.fixture(scope="module")
def mock_server():
    import subprocess
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "_build/liboracle_mock.so"], check=True)
    lib = C.CDLL(str(MOCK))
    lib.oracle_mock_serve_start.restype = C.c_int
    lib.oracle_mock_serve_start.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t]
    err = C.create_string_buffer(512)
    port = lib.oracle_mock_serve_start(CFG.encode(), b"127.0.0.1:0", err, 512)
    assert port > 0, err.value
    yield port
    lib.oracle_mock_serve_stop()


def test_health_reports_every_stage(mock_server):
    st, ctype, body = call(mock_server, "GET", "/v1/health")
    assert st == 200 and ctype == "application/json"
    assert json.loads(body) == {"thinker": "UP", "talker": "UP", "vocoder": "UP"}


def test_bad_requests_are_400(mock_server):
    assert call(mock_server, "POST", "/v1/generate", {"prompt_tokens": []})[0] == 400
    assert call(mock_server, "POST", "/v1/generate", "{not json")[0] == 400
    assert call(mock_server, "POST", "/v1/generate", {"prompt_tokens": [0, 300]})[0] == 400
    assert call(mock_server, "GET", "/v1/generate")[0] == 405
    assert call(mock_server, "GET", "/nope")[0] == 404


def test_non_streaming_matches_the_oracle(mock_server):
    import oracle
    st, _, body = call(mock_server, "POST", "/v1/generate", {"request_id": 501, "prompt_tokens": [1, 2, 3], "seed": 5})
    assert st == 200, body
    j = json.loads(body)
    text, hidden = oracle.thinker_generate([1, 2, 3], 5)
    codec = oracle.talker_generate(text, hidden)
    assert j["text_tokens"] == text
    assert j["codec_tokens"] == codec
    assert b64_i32(j["waveform_b64"]) == oracle.denoise_closed_form(codec, 16)
    assert "jct_us" in j["metrics"] and j["metrics"]["status"] == "DONE"


def test_streaming_is_ndjson_ending_in_done(mock_server):
    import oracle
    st, ctype, body = call(mock_server, "POST", "/v1/generate",
                           {"request_id": 502, "prompt_tokens": [9, 8, 7], "seed": 1, "stream": True})
    assert st == 200 and ctype == "application/x-ndjson"
    frames = [json.loads(l) for l in body.splitlines() if l]
    assert len(frames) >= 2
    wave = []
    for i, f in enumerate(frames[:-1]):
        assert f["type"] == "waveform_chunk" and f["seq"] == i
        wave += b64_i32(f["data_b64"])
    assert frames[-1]["type"] == "done" and "metrics" in frames[-1]
    text, hidden = oracle.thinker_generate([9, 8, 7], 1)
    assert wave == oracle.denoise_closed_form(oracle.talker_generate(text, hidden), 16)


def test_aggregate_metrics_count_completions(mock_server):
    assert call(mock_server, "POST", "/v1/generate", {"request_id": 503, "prompt_tokens": [4], "seed": 2})[0] == 200
    st, _, body = call(mock_server, "GET", "/v1/metrics")
    assert st == 200 and json.loads(body)["requests_done"] >= 1


@pytest.mark.gpu
def test_b200_pipeline_serves_http_streaming_and_plain():
    from paper_2602_02204_b200.serve import Pipeline
    p = Pipeline(CFG, weight_seed=1234, small_models=True, device=0)
    port = p.serve_start("127.0.0.1:0")
    try:
        assert json.loads(call(port, "GET", "/v1/health")[2]) == {"thinker": "UP", "talker": "UP", "vocoder": "UP"}
        st, _, body = call(port, "POST", "/v1/generate", {"request_id": 7, "prompt_tokens": [5, 6, 7, 8], "seed": 3})
        assert st == 200, body
        plain = json.loads(body)
        assert len(plain["codec_tokens"]) == 4 * len(plain["text_tokens"])
        wave_plain = b64_i32(plain["waveform_b64"])
        assert len(wave_plain) == 16 * len(plain["codec_tokens"])
        # the DiT noise is keyed by (request id, position, sample): replay the SAME
        # request id streamed on a fresh orchestrator
        p.serve_stop()
        port = p.serve_start("127.0.0.1:0")
        st, ctype, body = call(port, "POST", "/v1/generate",
                               {"request_id": 7, "prompt_tokens": [5, 6, 7, 8], "seed": 3, "stream": True})
        assert st == 200 and ctype == "application/x-ndjson"
        frames = [json.loads(l) for l in body.splitlines() if l]
        assert frames[-1]["type"] == "done"
        wave = [s for f in frames[:-1] for s in b64_i32(f["data_b64"])]
        assert [f["seq"] for f in frames[:-1]] == list(range(len(frames) - 1))
        # greedy, batch-invariant device models: the same prompt gives the same waveform
        assert wave == wave_plain
        assert json.loads(call(port, "GET", "/v1/metrics")[2])["requests_done"] >= 1
    finally:
        p.serve_stop()
        p.close()
