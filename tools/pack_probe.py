"""Connector pack kernel (K5) at synthetic large sizes:
64 sequences x 64 hidden rows x d = 2048 packed into FIX16 blobs in one launch
(16.8 MB of payload), plus the production size (one chunk of 4 rows).

  python tools/pack_probe.py [reps]

Prints one JSON line per size: kernel time from CUDA events around `reps`
back-to-back packs on the Thinker's stream (host-timed bracket, synchronised),
and algorithmic bytes = rows x d x 2 read + blob bytes written."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_02204_b200 import dev as D  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    m = D.model_default(D.THINKER)
    st = D.Stage(m, D.StageLimits(256, 64, 256, 0, 64), seed=3)
    n_seq, d = 64, m.d_model
    ids = list(range(1, n_seq + 1))
    for i in range(0, n_seq, 16):  # make the sequences resident (their hidden rings exist)
        grp = ids[i:i + 16]
        st.ar_step(grp, [D.PREFILL] * len(grp), [1] * len(grp), [0] * len(grp), [-1] * len(grp), [5] * len(grp))
    for rows, n_chunks in ((4, 1), (64, 8), (64, n_seq)):
        nb = D.pack_bytes(rows, d)
        stride = (nb + 15) // 16 * 16
        arena = D.mem_alloc(stride * n_chunks)
        seqs = ids[:n_chunks]
        args = (seqs, [0] * n_chunks, [rows] * n_chunks, [7] * (rows * n_chunks), arena,
                [c * stride for c in range(n_chunks)])
        for _ in range(3):
            st.pack_hidden(*args)
        st.wait()
        D.sync()
        t0 = time.perf_counter()
        for _ in range(reps):
            st.pack_hidden(*args)
        st.wait()
        D.sync()
        us = (time.perf_counter() - t0) / reps * 1e6
        algo = n_chunks * (rows * d * 2 + nb)
        print(json.dumps({"chunks": n_chunks, "rows_per_chunk": rows, "payload_MB": round(n_chunks * nb / 1e6, 3),
                          "us_per_launch_host_bracket": round(us, 2), "algo_bytes": algo,
                          "GBps": round(algo / us / 1e3, 1)}), flush=True)
        D.mem_free(arena)
    st.close()


if __name__ == "__main__":
    main()
