"""BASELINE.json configs 1-5 at full model size on one GPU: requests/s and
mean / p99 JCT of gen_workload(n, seed 7) in a closed loop (device clock).

  python tools/config_sweep.py [n] [concurrency]

One JSON line per config. Configs 2 and 4 name cross-GPU placements (stages
on separate GPUs / a replicated Talker); on a one-GPU box they run with every
stage on cuda:0 and, for config 4, the §8(e) 4-GPU placement folded onto the
one device (replicas with their own streams and KV pools)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200.serve import Pipeline  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
CONFIGS = [
    ("1 single AR stage", "thinker_only.json", None),
    ("2 Thinker->Talker", "thinker_talker.json", None),
    ("3 AR->DiT", "ar_dit.json", None),
    ("4 Thinker->Talker->Code2Wav", "omni3.json", None),
    ("4 ... Talker x2 (folded 4-GPU placement)", "omni3.json",
     {"thinker": "cuda:0", "talker": "cuda:0,cuda:0", "vocoder": "cuda:0"}),
    ("5 Ming-style branching", "ming_branch.json", None),
]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    conc = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    for name, cfg, placement in CONFIGS:
        c = json.loads((ROOT / "configs" / cfg).read_text())
        if placement:
            c["placement"] = placement
        p = Pipeline(json.dumps(c), weight_seed=7)
        p.bench(n=min(n, 32), seed=7, concurrency=conc, clock="device")  # warm-up: graphs, pools
        r = p.bench(n=n, seed=7, concurrency=conc, clock="device")
        p.close()
        print(json.dumps({"config": name, "file": cfg, "n": n, "concurrency": conc, "completed": r["completed"],
                          "requests_per_s": round(r["requests_per_s"], 2), "mean_jct_ms": round(r["mean_jct_us"] / 1e3, 2),
                          "p99_jct_ms": round(r["p99_jct_us"] / 1e3, 2), "text_tokens": r["text_tokens"],
                          "codec_tokens": r["codec_tokens"], "wave_samples": r["wave_samples"]}), flush=True)


if __name__ == "__main__":
    main()
