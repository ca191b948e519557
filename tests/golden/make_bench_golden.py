"""Bench-scale parity goldens, generated HERE with the reference itself
(oracle/_ref/libpmklc_ref.so = /root/reference/proj/core compiled from its own
sources). TEST INFRASTRUCTURE: tests/test_gpu_parity_scale.py compares the
B200 containers of the benchmark workloads against these numbers.

  config3  the exact bench.py default workload: 100 MB synthetic genome
           (synth genome, seed 2025, 10 segments), W=128, seeded untrained
           SPuM (k=3, t=32, scale 4, seed 0xACE3), CompressConfig defaults
           (s=k=3, t=32, bs=320, smp 0.05, seed 42) -> flags 5. The reference
           compress() runs the whole input (128 chunk threads); recorded:
           container length + FNV-1a, every chunk's payload FNV-1a, inbound
           snapshot hash (WorkerStats::snapshot_recv_hash) and early loss.
  sprm     the SPrM pre-pass (pretrain_private, training.cpp:62-83) at the
           default widths on the first 3.2 MB of the same genome (> 3,000
           strictly sequential Adam steps, warm-started from the SPuM as
           compress() does), and the whole flags-6 container of that prefix
           at W=4 (selector_threshold 0).

Usage: python tests/golden/make_bench_golden.py config3|sprm  (minutes to an
hour of CPU; the results are committed as tests/golden/bench_*.json).
"""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import oracles as O  # noqa: E402


def fnv(b: bytes) -> str:
    h = 0xcbf29ce484222325
    for x in b:
        h = ((h ^ x) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "config3"
    R = O.ref()
    tmp = Path(tempfile.mkdtemp(prefix="pmklc_golden_"))
    spum = str(tmp / "spum_k3_t32_s4.bin")
    fp = O.write_spum(spum, 3, 32, 4, 0xACE3)
    if what == "config3":
        n = 100_000_000
        raw = R.synth("genome", n, 2025, 10)
        cfg = O.make_cfg(workers=128, pub_path=spum)
        t0 = time.time()
        blob, st = R.compress(raw, cfg, with_stats=True)
        dt = time.time() - t0
        hdr = O.parse_container(blob)
        chunks = []
        for i, (ts, tl, po, pl, trl) in enumerate(hdr["chunks"]):
            chunks.append({"token_start": ts, "token_len": tl, "payload_len": pl,
                           "payload_fnv": fnv(blob[po:po + pl]),
                           "recv_hash": f"{st[i].snapshot_recv_hash:016x}",
                           "sent_hash": f"{st[i].snapshot_sent_hash:016x}",
                           "early_loss_bits": st[i].early_loss_bits})
        out = {"workload": "bench.py config3 default: synth genome 100e6 B seed 2025 10 segments, "
                           "W=128, SPuM seed 0xACE3 (k3 t32 scale4, 2 layers), defaults",
               "input_fnv": fnv(raw[:1 << 20]) + " (first MiB)", "spum_fingerprint": f"{fp:016x}",
               "flags": hdr["flags"], "container_len": len(blob), "container_fnv": fnv(blob),
               "bits_per_base": 8.0 * len(blob) / n, "chunks": chunks,
               "reference_compress_s": dt, "reference_threads": os.cpu_count()}
        (HERE / "bench_config3.json").write_text(json.dumps(out, indent=1))
    elif what == "sprm":
        import numpy as np
        n = 3_200_000
        raw = R.synth("genome", 100_000_000, 2025, 10)[:n]
        codes = np.frombuffer(raw, np.uint8)
        codes = (((codes >> 1) ^ (codes >> 2)) & 3).astype(np.uint8).tobytes()
        tok, _ = R.skmer_encode(codes, 3, 3)
        # sprm_seed = second draw of Rng(seed=42) (pipeline.cpp:305-307)
        def splitmix(seed, k):
            s = seed
            out = []
            for _ in range(k):
                s = (s + 0x9e3779b97f4a7c15) & 0xFFFFFFFFFFFFFFFF
                z = s
                z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & 0xFFFFFFFFFFFFFFFF
                z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & 0xFFFFFFFFFFFFFFFF
                out.append(z ^ (z >> 31))
            return out
        dm_seed, sprm_seed = splitmix(42, 2)
        t0 = time.time()
        blob_model = R.pretrain_private(tok, 3, 32, 320, 4, sprm_seed, pub_path=spum)
        t_pre = time.time() - t0
        t0 = time.time()
        cont = R.compress(raw, O.make_cfg(workers=4, pub_path=spum, threshold=0))
        t_c = time.time() - t0
        hdr = O.parse_container(cont)
        assert hdr["priv"] == blob_model, "compress() pre-pass differs from pretrain_private()"
        steps = (len(tok) - 32 + 319) // 320
        out = {"workload": "first 3.2e6 B of the config3 genome; pretrain_private at scale 4, "
                           "bs 320, t 32, warm start from the SPuM (seed 0xACE3); compress W=4 "
                           "threshold 0 (flags 6)",
               "tokens": len(tok), "train_steps": steps, "sprm_seed": f"{sprm_seed:016x}",
               "sprm_blob_len": len(blob_model), "sprm_blob_fnv": fnv(blob_model),
               "container_len": len(cont), "container_fnv": fnv(cont), "flags": hdr["flags"],
               "payload_fnv": [fnv(cont[po:po + pl]) for (_, _, po, pl, _) in hdr["chunks"]],
               "reference_pretrain_s": t_pre, "reference_compress_s": t_c}
        (HERE / "bench_sprm_prefix.json").write_text(json.dumps(out, indent=1))
    else:
        raise SystemExit(__doc__)


if __name__ == "__main__":
    main()
